# shifted-block walk: parity tests, narrow-N probe (col:2 at N=64, col:1 at N=32), ncu of variant 8 at N=128
mkdir -p gpurun_out/p79 /tmp/p79
timeout 1200 python -m pytest tests/test_gpu_scale.py -k "shifted" tests/test_gpu_baseline_shapes.py -k "shifted or stencil160" -x -q > gpurun_out/p79/pytest.log 2>&1; echo "exit $?" >> gpurun_out/p79/pytest.log
timeout 900 python tools/experiments/shifted_probe.py --ns 64 --points "row:8,col:2,r:1@256;row:8,col:4,r:1@256" --variants 4,3,8 --blocks 128 > gpurun_out/p79/shifted_n64.log 2>&1
timeout 900 python tools/experiments/shifted_probe.py --ns 32 --points "row:8,col:1,r:1@256;row:8,col:4,r:1@256" --variants 4,3,8 --blocks 128 > gpurun_out/p79/shifted_n32.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_row_shifted' --launch-skip 1 -c 1 -o /tmp/p79/cap_cfg4_v8 \
  python tools/ncu_traffic.py run --config 4 --point row:8,col:4,r:1 --p 256 --hw-variant 8 > gpurun_out/p79/cap.log 2>&1
python tools/ncu_traffic.py merge /tmp/p79/cap_cfg4_v8.ncu-rep --config 4 --point row:8,col:4,r:1 --hw-variant 8 \
  --summary gpurun_out/p79/r02_ncu_cfg4_v8.json >> gpurun_out/p79/cap.log 2>&1
cp /tmp/p79/cap_cfg4_v8.ncu-rep gpurun_out/p79/ 2>/dev/null
cp profiles/ncu_traffic.json gpurun_out/p79/ncu_traffic.json
tail -3 gpurun_out/p79/pytest.log; grep -v Warn gpurun_out/p79/shifted_n64.log gpurun_out/p79/shifted_n32.log | grep -v "bitwise-equal-to-first True"; tail -3 gpurun_out/p79/cap.log
