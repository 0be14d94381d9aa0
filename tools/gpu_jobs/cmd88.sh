# sanitizer cases as a plain oracle-checked run (compute-sanitizer is closed on the pool) + selector regret at HEAD
mkdir -p gpurun_out/p88
timeout 900 python tools/sanitize_cases.py > gpurun_out/p88/cases.log 2>&1; echo "rc=$?" >> gpurun_out/p88/cases.log
timeout 2400 python tools/selector_regret.py --out gpurun_out/p88/r02_selector_regret_full.json > gpurun_out/p88/regret.log 2>&1
timeout 2400 python tools/selector_regret.py --holdout --out gpurun_out/p88/r02_selector_regret_holdout.json > gpurun_out/p88/regret_holdout.log 2>&1
grep -v Warn gpurun_out/p88/cases.log | tail -4; tail -n 2 gpurun_out/p88/regret.log gpurun_out/p88/regret_holdout.log | cut -c1-300
