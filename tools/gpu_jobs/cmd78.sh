# shifted-block walk: pair-pipelined pieces (9, 13) and occupancy (12) vs 8 and the warp-per-row walk
mkdir -p gpurun_out/p78
timeout 900 python tools/experiments/shifted_probe.py --ns 128,256 --points "row:4,col:4,r:1@256" --variants 4,8,9,12,13 --blocks 128,64,256 > gpurun_out/p78/shifted_cfg4.log 2>&1
grep -v Warn gpurun_out/p78/shifted_cfg4.log | grep -v "bitwise-equal-to-first True"
