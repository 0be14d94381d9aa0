"""The drop-in boundary from plain C (examples/c_abi_spmm.c): it compiles and
links against libsgap.so + the CUDA runtime with only include/sgap.h (CPU),
and on the B200 runs four Sgap families through sgap_run within 1e-5 of a
host double-precision product (GPU)."""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CUDA = Path("/usr/local/cuda")


def _build(tmp_path) -> Path:
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib_dir = ROOT / "paper_2209_02882_b200"
    if not (lib_dir / "libsgap.so").exists():
        pytest.skip("libsgap.so not built")
    exe = tmp_path / "c_abi_spmm"
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", str(ROOT / "include"), "-I", str(CUDA / "include"),
           str(ROOT / "examples" / "c_abi_spmm.c"), "-L", str(lib_dir), "-lsgap",
           "-L", str(CUDA / "lib64"), "-lcudart", f"-Wl,-rpath,{lib_dir}", "-lm", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_c_example_runs_on_device(tmp_path):
    out = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("OK")
