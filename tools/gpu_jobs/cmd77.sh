# shifted-block RB walk (row-multiple variants 8/9) vs the warp-per-row walk on config 4
mkdir -p gpurun_out/p77
timeout 900 python tools/experiments/shifted_probe.py --ns 128,256,512 --check > gpurun_out/p77/shifted_cfg4.log 2>&1
cat gpurun_out/p77/shifted_cfg4.log | grep -v Warn
