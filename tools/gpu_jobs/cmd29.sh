python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt29.log 2>&1; echo rc=$? >> gpurun_out/gt29.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke29.log 2>&1; echo rc=$? >> gpurun_out/smoke29.log
python bench.py --impl reference > gpurun_out/ref29.json 2> gpurun_out/ref29.err
python bench.py > gpurun_out/b29.json 2> gpurun_out/b29.err
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py > gpurun_out/san29_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/san29_$tool.log
done
