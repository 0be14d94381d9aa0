mkdir -p gpurun_out/p61
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/p61/san_$t.log 2>&1; echo rc=$? >> gpurun_out/p61/san_$t.log
done
( time timeout 1500 python bench.py ) > gpurun_out/p61/bench.json 2> gpurun_out/p61/bench.err
for t in memcheck racecheck synccheck; do tail -n 4 gpurun_out/p61/san_$t.log; done
cat gpurun_out/p61/bench.json | head -c 600; tail -n 4 gpurun_out/p61/bench.err
