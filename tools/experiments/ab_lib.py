"""A/B-time one point with the in-tree libsgap.so vs an alternative build
(SGAP_LIB env var points _native at it).  Usage: python ab_lib.py <config> <point> <variant>"""
import os
import subprocess
import sys

cfg, point, var = sys.argv[1], sys.argv[2], sys.argv[3]
for label, env in (("in-tree", {}), ("alt", {"SGAP_LIB": "tools/experiments/alt/libsgap.so"})):
    out = subprocess.run([sys.executable, "tools/kbench.py", "--config", cfg, "--points", point,
                          "--variants", var, "--reps", "9"], capture_output=True, text=True,
                         env={**os.environ, **env})
    print(label, [l for l in out.stdout.splitlines() if " ms " in l and "cuSPARSE" not in l])
