mkdir -p gpurun_out/p66
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "row_staged" > gpurun_out/p66/test.log 2>&1; echo rc=$? >> gpurun_out/p66/test.log
timeout 900 python tools/kbench.py --config 4 --n 256 --points "row:8,col:4,r:1@256;row:4,col:4,r:1@256;row:16,col:4,r:1@256;nnz:128,col:4,r:1@1024;row:32,col:4,r:1@1024" --variants 0,1,4 --reps 5 --check > gpurun_out/p66/cfg4_n256.log 2>&1
timeout 900 python tools/kbench.py --config 4 --n 512 --points "row:8,col:4,r:1@256;row:4,col:4,r:1@256;nnz:64,col:4,r:1@1024;row:32,col:4,r:1@256" --variants 0,1,4 --reps 5 --check > gpurun_out/p66/cfg4_n512.log 2>&1
tail -n 2 gpurun_out/p66/test.log; grep -v Warn gpurun_out/p66/cfg4_n256.log | head -8; grep -v Warn gpurun_out/p66/cfg4_n512.log | head -8
