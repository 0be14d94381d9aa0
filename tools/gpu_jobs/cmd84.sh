# sub-warp shifted-block walk (variant 8 at N/c = 16 / 8) vs the sub-warp walk (variant 4)
mkdir -p gpurun_out/p84
timeout 900 python tools/experiments/shifted_probe.py --ns 64,32 --points "row:8,col:4,r:1@256" --variants 4,8 --blocks 128,256 --check > gpurun_out/p84/shifted_sub.log 2>&1
grep -v Warn gpurun_out/p84/shifted_sub.log
