# final: config-4 N sweep with the slab form, HEAD ncu capture of the config-4 walk, full gated GPU suite + smoke
mkdir -p gpurun_out/p94 /tmp/p94
for n in 16 32 64 128 256 512; do
  timeout 1200 python tools/kbench.py --config 4 --n $n --all --reps 3 --out gpurun_out/p94/sweep_cfg4_n$n.json > gpurun_out/p94/sweep_cfg4_n$n.log 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_row_shifted' --launch-skip 1 -c 1 -o /tmp/p94/cap_cfg4_v8 \
  python tools/ncu_traffic.py run --config 4 --point row:8,col:4,r:1 --p 256 --hw-variant 8 > gpurun_out/p94/cap.log 2>&1
python tools/ncu_traffic.py merge /tmp/p94/cap_cfg4_v8.ncu-rep --config 4 --point row:8,col:4,r:1 --hw-variant 8 \
  --summary gpurun_out/p94/r02_ncu_cfg4_v8_slab.json >> gpurun_out/p94/cap.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/p94/ncu_traffic.json
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/p94/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/p94/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/p94/smoke.log 2>&1
python tools/sweep_table.py gpurun_out/p94/sweep_cfg4_n*.json; tail -1 gpurun_out/p94/cap.log; tail -2 gpurun_out/p94/pytest_gpu.log; tail -1 gpurun_out/p94/smoke.log
