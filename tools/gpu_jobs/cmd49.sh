mkdir -p gpurun_out/p49
timeout 600 python tools/experiments/panel_probe.py --config 3 --n 256 --panels 128,64,32 --variant 1 > gpurun_out/p49/cfg3_n256.log 2>&1
timeout 600 python tools/experiments/panel_probe.py --config 2 --n 128 --panels 64,32 --variant 5 > gpurun_out/p49/cfg2_n128.log 2>&1
timeout 900 python tools/experiments/panel_probe.py --config 5 --n 128 --panels 64,32 --variant 9 --rounds 3 > gpurun_out/p49/cfg5_n128.log 2>&1
tail -n 5 gpurun_out/p49/*.log
