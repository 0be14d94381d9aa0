mkdir -p gpurun_out/p58
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "row_blocked" > gpurun_out/p58/test.log 2>&1; echo rc=$? >> gpurun_out/p58/test.log
for n in 128 64; do
  c=$((n/32))
  timeout 900 python tools/kbench.py --config 4 --n $n --points "row:8,col:$c,r:1@256;row:4,col:$c,r:1@256;row:16,col:$c,r:1@256" --variants 4,6,7 --reps 5 --check > gpurun_out/p58/blk_cfg4_n$n.log 2>&1
done
tail -n 2 gpurun_out/p58/test.log; grep -v Warn gpurun_out/p58/blk_cfg4_n128.log | head -12
