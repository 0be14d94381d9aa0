# shifted-block walk at narrow N (col:2 at N=64, col:1 at N=32) and the variant-8 ncu summary
mkdir -p gpurun_out/p80 /tmp/p80
timeout 900 python tools/experiments/shifted_probe.py --ns 64 --points "row:8,col:2,r:1@256;row:8,col:4,r:1@256" --variants 4,3,8 --blocks 128 > gpurun_out/p80/shifted_n64.log 2>&1
timeout 900 python tools/experiments/shifted_probe.py --ns 32 --points "row:8,col:1,r:1@256;row:8,col:4,r:1@256" --variants 4,3,8 --blocks 128 > gpurun_out/p80/shifted_n32.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_row_shifted' --launch-skip 1 -c 1 -o /tmp/p80/cap_cfg4_v8 \
  python tools/ncu_traffic.py run --config 4 --point row:8,col:4,r:1 --p 256 --hw-variant 8 > gpurun_out/p80/cap.log 2>&1
python tools/ncu_traffic.py merge /tmp/p80/cap_cfg4_v8.ncu-rep --config 4 --point row:8,col:4,r:1 --hw-variant 8 \
  --summary gpurun_out/p80/r02_ncu_cfg4_v8.json >> gpurun_out/p80/cap.log 2>&1
ncu -i /tmp/p80/cap_cfg4_v8.ncu-rep --page source --csv > /tmp/p80/src.csv 2>/dev/null; head -c 3000000 /tmp/p80/src.csv > gpurun_out/p80/src_head.csv
cp profiles/ncu_traffic.json gpurun_out/p80/ncu_traffic.json
grep -v Warn gpurun_out/p80/shifted_n64.log gpurun_out/p80/shifted_n32.log | grep -v "bitwise-equal-to-first True"; tail -3 gpurun_out/p80/cap.log
