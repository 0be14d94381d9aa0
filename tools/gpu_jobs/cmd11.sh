timeout 1200 python tools/experiments/cold_hint_probe.py --config 5 > gpurun_out/coldhint_cfg5.log 2>&1
timeout 600 python tools/experiments/cold_hint_probe.py --config 2 --hot 8192,16384,32768,65536,131072 > gpurun_out/coldhint_cfg2.log 2>&1
KR='regex:^(k_nnz_multiple)$'
mkdir -p gpurun_out/prof11; cp profiles/ncu_traffic.json gpurun_out/prof11/
for v in 5 1; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "$KR" --launch-skip 1 -c 1 -f -o /tmp/cap_cfg5_v$v python tools/ncu_traffic.py run --config 5 --point nnz:512,col:4,r:1 --p 256 --hw-variant $v > gpurun_out/prof11/cap_v$v.log 2>&1
  python tools/ncu_traffic.py merge /tmp/cap_cfg5_v$v.ncu-rep --config 5 --point nnz:512,col:4,r:1 --hw-variant $v --summary gpurun_out/prof11/r02_ncu_cfg5_v$v.json >> gpurun_out/prof11/status.txt 2>&1
done
for v in 5 1; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "$KR" --launch-skip 1 -c 1 -f -o /tmp/cap_cfg2_v$v python tools/ncu_traffic.py run --config 2 --point nnz:512,col:4,r:1 --p 256 --hw-variant $v > gpurun_out/prof11/cap2_v$v.log 2>&1
  python tools/ncu_traffic.py merge /tmp/cap_cfg2_v$v.ncu-rep --config 2 --point nnz:512,col:4,r:1 --hw-variant $v --summary gpurun_out/prof11/r02_ncu_cfg2_v$v.json >> gpurun_out/prof11/status.txt 2>&1
done
cp profiles/ncu_traffic.json gpurun_out/prof11/ncu_traffic.json
