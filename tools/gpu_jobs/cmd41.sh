KR='regex:^(k_nnz_multiple)$'
mkdir -p gpurun_out/prof41; cp profiles/ncu_traffic.json gpurun_out/prof41/
timeout 900 ncu --set full --clock-control none --import-source on -k "$KR" --launch-skip 1 -c 1 -f -o /tmp/cap41 python tools/ncu_traffic.py run --config 5 --point nnz:512,col:4,r:1 --p 256 --hw-variant 9 > gpurun_out/prof41/cap.log 2>&1
python tools/ncu_traffic.py merge /tmp/cap41.ncu-rep --config 5 --point nnz:512,col:4,r:1 --hw-variant 9 --summary gpurun_out/prof41/r02_ncu_final_cfg5_v9.json >> gpurun_out/prof41/status.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/prof41/ncu_traffic.json
