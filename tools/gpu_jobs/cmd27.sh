timeout 2400 python tools/selector_regret.py --out gpurun_out/r02_selector_regret_full.json > gpurun_out/regret27.log 2>&1
