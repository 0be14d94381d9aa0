python -m pytest tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "row_staged" > gpurun_out/gt21.log 2>&1; echo rc=$? >> gpurun_out/gt21.log
for n in 32 64 128; do
  c=$((n/32))
  timeout 900 python tools/kbench.py --config 4 --n $n --points "row:8,col:$c,r:1@256;row:4,col:$c,r:1@256;row:16,col:$c,r:1@256;row:2,col:$c,r:1@256" --variants 4,8 --reps 7 > gpurun_out/pf_cfg4_n$n.log 2>&1
done
