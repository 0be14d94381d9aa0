# sub-warp shifted walk restricted to N/c = 16: parity tests (bitwise vs variant 4, config 4 sweep, selector)
mkdir -p gpurun_out/p85
timeout 1500 python -m pytest tests/test_gpu_scale.py tests/test_gpu_baseline_shapes.py tests/test_gpu_parity.py -x -q > gpurun_out/p85/pytest.log 2>&1; echo "exit $?" >> gpurun_out/p85/pytest.log
tail -3 gpurun_out/p85/pytest.log
