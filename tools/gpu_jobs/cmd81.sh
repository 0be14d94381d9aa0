# shifted-block walk: L1 prefetch of the next piece's B rows (variant 12, experiment) vs 8
mkdir -p gpurun_out/p81
timeout 900 python tools/experiments/shifted_probe.py --ns 128,256 --points "row:8,col:4,r:1@256" --variants 8,12,9 --blocks 128,64 --rounds 7 > gpurun_out/p81/shifted_pf.log 2>&1
grep -v Warn gpurun_out/p81/shifted_pf.log | grep -v "bitwise-equal-to-first True"
