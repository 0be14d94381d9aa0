# compute-sanitizer with the shifted-block walk cases (memcheck / racecheck / synccheck)
mkdir -p gpurun_out/p87
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/p87/$tool.log 2>&1; echo "rc=$?" >> gpurun_out/p87/$tool.log
done
for tool in memcheck racecheck synccheck; do echo "## $tool"; grep -v Warn gpurun_out/p87/$tool.log | tail -4; done
