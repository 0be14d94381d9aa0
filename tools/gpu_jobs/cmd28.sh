timeout 2400 python tools/selector_regret.py --holdout --out gpurun_out/r02_selector_regret_holdout.json > gpurun_out/regret28.log 2>&1
