mkdir -p gpurun_out/p60
timeout 900 python tools/kbench.py --config 4 --n 128 --points "row:8,col:4,r:1@256;row:4,col:4,r:1@256;row:2,col:4,r:1@256" --variants 4,6,7 --reps 5 --check > gpurun_out/p60/blk_cfg4_n128.log 2>&1
grep -v Warn gpurun_out/p60/blk_cfg4_n128.log | head -12
