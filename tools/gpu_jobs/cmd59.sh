mkdir -p gpurun_out/p59 /tmp/p59
for v in 6 4; do
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'^(k_row_blocked|k_row_staged)$' --launch-skip 1 -c 1 -o /tmp/p59/cfg4_v$v \
  python tools/ncu_traffic.py run --config 4 --n 128 --point row:4,col:4,r:1 --p 256 --hw-variant $v > gpurun_out/p59/run_v$v.log 2>&1
ncu -i /tmp/p59/cfg4_v$v.ncu-rep --page raw --csv > gpurun_out/p59/raw_v$v.csv
ncu -i /tmp/p59/cfg4_v$v.ncu-rep --page details --csv > gpurun_out/p59/details_v$v.csv
ncu -i /tmp/p59/cfg4_v$v.ncu-rep --page source --csv --print-source sass > gpurun_out/p59/sass_v$v.csv 2>&1
done
ls -la gpurun_out/p59
