mkdir -p gpurun_out/sw48
timeout 2400 python tools/kbench.py --config 5 --n 128 --all --reps 2 --out gpurun_out/sw48/sweep_cfg5_n128.json > gpurun_out/sw48/sweep_cfg5_n128.log 2>&1
timeout 1200 python tools/kbench.py --config 3 --n 256 --all --reps 3 --out gpurun_out/sw48/sweep_cfg3_n256.json > gpurun_out/sw48/sweep_cfg3_n256.log 2>&1
