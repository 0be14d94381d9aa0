# float64 (the reference's default precision, sim.run(precision="double")) on the BASELINE workloads
mkdir -p gpurun_out/p75
timeout 900 python tools/kbench.py --dtype f64 --config 2 --n 128 --points "nnz:512,col:4,r:1@256;nnz:256,col:4,r:1@256;nnz:512,col:2,r:1@256;nnz:128,col:2,r:1@1024" --variants 1,5,2 --reps 3 --check > gpurun_out/p75/cfg2.log 2>&1
timeout 900 python tools/kbench.py --dtype f64 --config 3 --n 64 --points "nnz:512,col:4,r:1@256;nnz:512,col:2,r:1@256;nnz:256,col:2,r:1@1024" --variants 1,5,2 --reps 3 --check > gpurun_out/p75/cfg3.log 2>&1
timeout 900 python tools/kbench.py --dtype f64 --config 4 --n 128 --points "row:8,col:4,r:1@256;row:8,col:2,r:1@256;row:4,col:2,r:1@256;nnz:256,col:2,r:1@1024" --variants 0,2,4,1 --reps 3 --check > gpurun_out/p75/cfg4.log 2>&1
for c in 2 3 4; do grep -v Warn gpurun_out/p75/cfg$c.log | head -6; grep -c " OK" gpurun_out/p75/cfg$c.log; grep FAIL gpurun_out/p75/cfg$c.log; done; true
