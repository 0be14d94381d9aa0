# HEAD ncu capture of the config-4 shifted walk (64-thread CTAs) for roofline.traffic
mkdir -p gpurun_out/p92 /tmp/p92
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_row_shifted' --launch-skip 1 -c 1 -o /tmp/p92/cap_cfg4_v8 \
  python tools/ncu_traffic.py run --config 4 --point row:8,col:4,r:1 --p 256 --hw-variant 8 > gpurun_out/p92/cap.log 2>&1
python tools/ncu_traffic.py merge /tmp/p92/cap_cfg4_v8.ncu-rep --config 4 --point row:8,col:4,r:1 --hw-variant 8 \
  --summary gpurun_out/p92/r02_ncu_cfg4_v8_head.json >> gpurun_out/p92/cap.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/p92/ncu_traffic.json
tail -2 gpurun_out/p92/cap.log
