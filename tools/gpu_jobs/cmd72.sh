mkdir -p gpurun_out/p72
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "row_staged" > gpurun_out/p72/test.log 2>&1; echo rc=$? >> gpurun_out/p72/test.log
timeout 900 python tools/kbench.py --config 4 --n 16 --points "row:8,col:4,r:1@256;row:4,col:4,r:1@256;row:16,col:4,r:1@256;row:8,col:2,r:1@1024" --variants 2,3,4 --reps 5 --check > gpurun_out/p72/cfg4_n16.log 2>&1
tail -n 2 gpurun_out/p72/test.log; grep -v Warn gpurun_out/p72/cfg4_n16.log | head -8; grep -c OK gpurun_out/p72/cfg4_n16.log
