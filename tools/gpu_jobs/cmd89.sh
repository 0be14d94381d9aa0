# shifted walk CTA size (default 64 vs 128), config-4 bench line, config-5 headline bench line at HEAD
mkdir -p gpurun_out/p89
timeout 900 python tools/experiments/shifted_probe.py --ns 64,128,256 --points "row:8,col:4,r:1@256" --variants 8 --blocks 0,128,32 --rounds 7 > gpurun_out/p89/blocks.log 2>&1
timeout 900 python bench.py --config 4 --no-cpu > gpurun_out/p89/bench_cfg4.json 2> gpurun_out/p89/bench_cfg4.err
timeout 1200 python bench.py > gpurun_out/p89/bench_cfg5.json 2> gpurun_out/p89/bench_cfg5.err
grep -v Warn gpurun_out/p89/blocks.log | grep -v "bitwise-equal-to-first True"; cut -c1-400 gpurun_out/p89/bench_cfg4.json gpurun_out/p89/bench_cfg5.json
