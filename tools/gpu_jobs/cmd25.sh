# final-build sweeps (every templated point and walk) + ncu captures of the picks
mkdir -p gpurun_out/sw25
for spec in "2 128" "3 64" "3 256" "4 16" "4 32" "4 64" "4 128" "4 256" "4 512"; do
  set -- $spec
  timeout 1200 python tools/kbench.py --config $1 --n $2 --all --reps 3 --out gpurun_out/sw25/sweep_cfg$1_n$2.json > gpurun_out/sw25/sweep_cfg$1_n$2.log 2>&1
done
KR='regex:^(k_nnz_multiple|k_row_staged)$'
mkdir -p gpurun_out/prof25; cp profiles/ncu_traffic.json gpurun_out/prof25/
for spec in "5 nnz:512,col:4,r:1 256 9" "3 nnz:512,col:4,r:1 256 1" "2 nnz:512,col:4,r:1 256 5"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k "$KR" --launch-skip 1 -c 1 -f -o /tmp/cap25_cfg$1 python tools/ncu_traffic.py run --config $1 --point $2 --p $3 --hw-variant $4 > gpurun_out/prof25/cap_cfg$1.log 2>&1
  python tools/ncu_traffic.py merge /tmp/cap25_cfg$1.ncu-rep --config $1 --point $2 --hw-variant $4 --summary gpurun_out/prof25/r02_ncu_final_cfg$1_v$4.json >> gpurun_out/prof25/status.txt 2>&1
done
cp profiles/ncu_traffic.json gpurun_out/prof25/ncu_traffic.json
