python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt5.log 2>&1; echo rc=$? >> gpurun_out/gt5.log
for cfg in 2 3 5; do
  timeout 900 python tools/kbench.py --config $cfg --points "nnz:512,col:4,r:1@256;nnz:256,col:4,r:1@256" --variants 1,5 --reps 7 > gpurun_out/ab_rp_cfg$cfg.log 2>&1
done
