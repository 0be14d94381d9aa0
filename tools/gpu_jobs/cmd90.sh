# sub-warp shifted walk at N/c = 8 (4 lane groups of 2 rows) vs the sub-warp walk
mkdir -p gpurun_out/p90
timeout 900 python tools/experiments/shifted_probe.py --ns 32,64 --points "row:8,col:4,r:1@256" --variants 4,8 --blocks 0,128 --rounds 7 --check > gpurun_out/p90/sub8.log 2>&1
grep -v Warn gpurun_out/p90/sub8.log
