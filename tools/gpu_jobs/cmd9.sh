KR='regex:^(k_nnz_multiple)$'
timeout 900 ncu --set full --clock-control none --import-source on -k "$KR" --launch-skip 1 -c 1 -f -o gpurun_out/cap_cfg2_v5 python tools/ncu_traffic.py run --config 2 --point nnz:512,col:4,r:1 --p 256 --hw-variant 5 > gpurun_out/cap9.log 2>&1
