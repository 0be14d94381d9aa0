timeout 1800 python tools/scaling_projection.py --strong --worlds 1,2,4,8 --variant 9 --out gpurun_out/r02_scaling_projection_strong.json > gpurun_out/scal22.log 2>&1
timeout 2400 python tools/selector_regret.py --out gpurun_out/r02_selector_regret.json > gpurun_out/regret22.log 2>&1
timeout 1200 python tools/refgen_bench.py --config 2 --out gpurun_out/r02_refgen_cfg2.json > gpurun_out/refgen22_cfg2.log 2>&1
