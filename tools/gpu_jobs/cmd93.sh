# shared-slab values in the shifted walks (default now), N/c = 8 enabled: parity + timings + config-4 bench line
mkdir -p gpurun_out/p93
timeout 1500 python -m pytest tests/test_gpu_scale.py tests/test_gpu_baseline_shapes.py -x -q > gpurun_out/p93/pytest.log 2>&1; echo "exit $?" >> gpurun_out/p93/pytest.log
timeout 900 python tools/experiments/shifted_probe.py --ns 32,64,128,256,512 --points "row:8,col:4,r:1@256" --variants 4,8 --blocks 0 --rounds 7 > gpurun_out/p93/probe.log 2>&1
timeout 900 python bench.py --config 4 --no-cpu > gpurun_out/p93/bench_cfg4.json 2> gpurun_out/p93/bench_cfg4.err
tail -2 gpurun_out/p93/pytest.log; grep -v Warn gpurun_out/p93/probe.log | grep -v "bitwise-equal-to-first True"; cut -c1-200 gpurun_out/p93/bench_cfg4.json
