python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "nnz_one_segment_walk or long_chunk_walks or zoo_every" > gpurun_out/gt16.log 2>&1; echo rc=$? >> gpurun_out/gt16.log
for cfg in 2 3 4; do
  timeout 900 python tools/kbench.py --config $cfg --points "nnz:1,col:4,r:8@1024;nnz:1,col:4,r:32@1024;nnz:1,col:4,r:4@256;nnz:1,col:4,r:1@256" --variants 0,1 --reps 5 > gpurun_out/nnzone_cfg$cfg.log 2>&1
done
