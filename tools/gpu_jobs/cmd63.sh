# HEAD captures for the bench's roofline.traffic and the launch list of the bench command
mkdir -p gpurun_out/p63 /tmp/p63
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'^(k_nnz_multiple)$' --launch-skip 1 -c 1 -o /tmp/p63/cap_cfg5_v9 \
  python tools/ncu_traffic.py run --config 5 --point nnz:512,col:4,r:1 --p 1024 --hw-variant 9 > gpurun_out/p63/cap.log 2>&1
python tools/ncu_traffic.py merge /tmp/p63/cap_cfg5_v9.ncu-rep --config 5 --point nnz:512,col:4,r:1 --hw-variant 9 \
  --summary gpurun_out/p63/r02_ncu_head_cfg5_v9.json >> gpurun_out/p63/cap.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/p63/ncu_traffic.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:sgap:: -c 400 --csv \
  --log-file gpurun_out/p63/launches_cfg5.csv python bench.py --steps 3 --warmup 3 --point nnz:512,col:4,r:1 --p 1024 --hw-variant 9 --no-e2e --no-cpu > gpurun_out/p63/b.json 2> gpurun_out/p63/b.err
tail -n 3 gpurun_out/p63/cap.log; wc -l gpurun_out/p63/launches_cfg5.csv
