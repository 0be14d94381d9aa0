# HEAD validation: gated GPU suite, smoke, default bench line
mkdir -p gpurun_out/p91
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/p91/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/p91/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/p91/smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/p91/bench.json 2> gpurun_out/p91/bench.err
tail -2 gpurun_out/p91/pytest_gpu.log; tail -1 gpurun_out/p91/smoke.log; cut -c1-300 gpurun_out/p91/bench.json
