# after the shifted-block walk: full gated GPU suite, float64 A/B on config 4, config-4 bench line
mkdir -p gpurun_out/p82
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/p82/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/p82/pytest_gpu.log
timeout 900 python tools/kbench.py --dtype f64 --config 4 --n 128 --points "row:8,col:2,r:1@256" --variants 4,8 --reps 5 --check > gpurun_out/p82/f64_cfg4.log 2>&1
timeout 900 python bench.py --config 4 --no-cpu --sweep gpurun_out/p82/sweep_cfg4.json > gpurun_out/p82/bench_cfg4.json 2> gpurun_out/p82/bench_cfg4.err
tail -3 gpurun_out/p82/pytest_gpu.log; grep -v Warn gpurun_out/p82/f64_cfg4.log | head -8; cut -c1-900 gpurun_out/p82/bench_cfg4.json
