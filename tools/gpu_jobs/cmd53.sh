mkdir -p gpurun_out/p53
timeout 600 python tools/experiments/panel_probe.py --config 3 --n 256 --panels 64,32 --variant 1 --rounds 6 > gpurun_out/p53/cfg3_n256.log 2>&1
tail -n 6 gpurun_out/p53/*.log
