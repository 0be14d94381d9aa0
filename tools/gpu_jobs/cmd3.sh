python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt3.log 2>&1; echo rc=$? >> gpurun_out/gt3.log
timeout 1200 python tools/experiments/hot_window_probe.py > gpurun_out/hotwin.log 2>&1
timeout 2400 python tools/dgsparse_grid.py --out gpurun_out/dgsparse.json > gpurun_out/dgsparse.log 2>&1
