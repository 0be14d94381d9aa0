# selector regret at the end-of-round build (new RB walks, column panels)
mkdir -p gpurun_out/p70
timeout 2400 python tools/selector_regret.py --out gpurun_out/p70/r02_selector_regret_full.json > gpurun_out/p70/regret.log 2>&1
timeout 2400 python tools/selector_regret.py --holdout --out gpurun_out/p70/r02_selector_regret_holdout.json > gpurun_out/p70/regret_holdout.log 2>&1
tail -n 3 gpurun_out/p70/regret.log gpurun_out/p70/regret_holdout.log
