python -m pytest tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "row_blocked" > gpurun_out/gt8.log 2>&1; echo rc=$? >> gpurun_out/gt8.log
for n in 32 64 128; do
  c=$((n/32))
  timeout 900 python tools/kbench.py --config 4 --n $n --points "row:8,col:$c,r:1@256;row:4,col:$c,r:1@256;row:16,col:$c,r:1@256;row:8,col:$c,r:1@1024" --variants 4,6,7 --reps 5 --check > gpurun_out/blk_cfg4_n$n.log 2>&1
done
