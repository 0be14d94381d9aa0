# end-of-round sweeps at the final build: every templated point and walk per BASELINE workload
mkdir -p gpurun_out/sw67
for spec in "2 128" "3 64" "3 256" "4 16" "4 32" "4 64" "4 128" "4 256" "4 512"; do
  set -- $spec
  timeout 1500 python tools/kbench.py --config $1 --n $2 --all --reps 3 --out gpurun_out/sw67/sweep_cfg$1_n$2.json > gpurun_out/sw67/sweep_cfg$1_n$2.log 2>&1
done
timeout 2400 python tools/kbench.py --config 5 --n 128 --all --reps 2 --out gpurun_out/sw67/sweep_cfg5_n128.json > gpurun_out/sw67/sweep_cfg5_n128.log 2>&1
ls gpurun_out/sw67; for f in gpurun_out/sw67/*.log; do echo $f; sed -n 2,3p $f; done
