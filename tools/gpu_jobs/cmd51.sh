mkdir -p gpurun_out/p51
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -k "panel or cold_column" > gpurun_out/p51/test.log 2>&1
timeout 600 python tools/experiments/ab_interleaved.py --config 3 --n 256 --variants 1,9,10 --rounds 5 > gpurun_out/p51/ab_cfg3_n256.log 2>&1
tail -n 3 gpurun_out/p51/test.log; tail -n 4 gpurun_out/p51/ab_*.log
