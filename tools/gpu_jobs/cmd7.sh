timeout 900 python tools/experiments/hot_window_probe.py --config 2 --hot 16384,32768,65536,131072 --hw-variant 5 > gpurun_out/hotwin_cfg2.log 2>&1
timeout 900 python tools/experiments/hot_window_probe.py --config 5 --hot 131072,163840 --hw-variant 1 > gpurun_out/hotwin_cfg5_rp.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san2_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san2_$tool.log
done
python bench.py > gpurun_out/b5_7.json 2> gpurun_out/b5_7.err
