# ncu --set full captures of the benched kernels (traffic for bench.py's roofline) + sanitizer runs
KR='regex:^(k_nnz_multiple|k_nnz_multiple_tma|k_nnz_multiple_staged|k_nnz_one|k_row_multiple|k_row_interleaved|k_row_staged|k_row_reciprocal)$'
mkdir -p gpurun_out/prof
cp profiles/ncu_traffic.json gpurun_out/prof/ 2>/dev/null
for spec in "5 nnz:512,col:4,r:1 256 1" "2 nnz:512,col:4,r:1 256 1" "3 nnz:512,col:4,r:1 256 1" "4 row:8,col:4,r:1 256 4"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k "$KR" --launch-skip 1 -c 1 -f -o /tmp/cap_cfg$1 python tools/ncu_traffic.py run --config $1 --point $2 --p $3 --hw-variant $4 > gpurun_out/prof/cap_cfg$1.log 2>&1
  echo "cfg$1 ncu rc=$?" >> gpurun_out/prof/status.txt
  python tools/ncu_traffic.py merge /tmp/cap_cfg$1.ncu-rep --config $1 --point $2 --hw-variant $4 --summary gpurun_out/prof/r02_ncu_cfg$1.json >> gpurun_out/prof/status.txt 2>&1
  ls -la /tmp/cap_cfg$1.ncu-rep >> gpurun_out/prof/status.txt
done
cp profiles/ncu_traffic.json gpurun_out/prof/ncu_traffic.json
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py > gpurun_out/prof/san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/prof/san_$tool.log
done
