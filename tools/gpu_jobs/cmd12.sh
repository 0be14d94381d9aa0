python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt12.log 2>&1; echo rc=$? >> gpurun_out/gt12.log
for cfg in 5 2; do
  timeout 900 python tools/kbench.py --config $cfg --points "nnz:512,col:4,r:1@256;nnz:256,col:4,r:1@256" --variants 1,5,9 --reps 7 > gpurun_out/ab12_cfg$cfg.log 2>&1
done
