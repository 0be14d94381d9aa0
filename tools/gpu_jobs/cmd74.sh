mkdir -p gpurun_out/p74
timeout 900 python tools/experiments/short_rows_probe.py --config 2 > gpurun_out/p74/cfg2.log 2>&1
timeout 900 python tools/experiments/short_rows_probe.py --config 5 > gpurun_out/p74/cfg5.log 2>&1
cat gpurun_out/p74/cfg2.log gpurun_out/p74/cfg5.log | grep -v Warn
