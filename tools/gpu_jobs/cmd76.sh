# HEAD validation after the container re-creation: gated GPU suite, smoke, bench line, reference arm
mkdir -p gpurun_out/p76
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/p76/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/p76/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/p76/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/p76/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/p76/bench.json 2> gpurun_out/p76/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/p76/bench_ref.json 2> gpurun_out/p76/bench_ref.err
tail -3 gpurun_out/p76/pytest_gpu.log; cat gpurun_out/p76/smoke.log | tail -2; cat gpurun_out/p76/bench.json gpurun_out/p76/bench_ref.json | cut -c1-600
