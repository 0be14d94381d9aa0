# float64 config 4 with the shared-slab shifted walk (reference default precision)
mkdir -p gpurun_out/p95
timeout 900 python tools/kbench.py --dtype f64 --config 4 --n 128 --points "row:8,col:2,r:1@256" --variants 4,8 --reps 5 --check > gpurun_out/p95/f64_cfg4.log 2>&1
grep -v Warn gpurun_out/p95/f64_cfg4.log | head -6
