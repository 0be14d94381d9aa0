# config 4 narrow-N sweeps with the sub-warp RB walk; sanitizers with the new row cases
mkdir -p gpurun_out/sw69 gpurun_out/p69
for spec in "4 16" "4 32" "4 64"; do
  set -- $spec
  timeout 1500 python tools/kbench.py --config $1 --n $2 --all --reps 3 --out gpurun_out/sw69/sweep_cfg$1_n$2.json > gpurun_out/sw69/sweep_cfg$1_n$2.log 2>&1
done
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/p69/san_$t.log 2>&1; echo rc=$? >> gpurun_out/p69/san_$t.log
done
for f in gpurun_out/sw69/*.log; do echo $f; sed -n 2,3p $f; done
for t in memcheck racecheck synccheck; do grep -v "^=========  " gpurun_out/p69/san_$t.log | tail -n 3; done
