mkdir -p gpurun_out/p62
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/p62/san_$t.log 2>&1; echo rc=$? >> gpurun_out/p62/san_$t.log
done
for t in memcheck racecheck synccheck; do grep -v "^=========  " gpurun_out/p62/san_$t.log | tail -n 6; done
