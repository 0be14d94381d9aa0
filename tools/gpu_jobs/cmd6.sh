for cfg in 2 5 3; do
  timeout 900 python tools/kbench.py --config $cfg --points "nnz:512,col:4,r:1@256;nnz:256,col:4,r:1@256" --variants 1,5 --reps 7 > gpurun_out/ab2_rp_cfg$cfg.log 2>&1
done
