mkdir -p gpurun_out/p73
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "row_staged" > gpurun_out/p73/test.log 2>&1; echo rc=$? >> gpurun_out/p73/test.log
timeout 900 python tools/kbench.py --config 4 --n 8 --points "row:1,col:4,r:1@256;row:4,col:4,r:1@256;row:8,col:4,r:1@256;row:4,col:2,r:1@256;row:1/2,col:4,r:2@256" --variants 0,2,4 --reps 5 --check > gpurun_out/p73/cfg4_n8.log 2>&1
timeout 900 python tools/kbench.py --config 4 --n 4 --points "row:1,col:4,r:1@256;row:4,col:2,r:1@256;row:8,col:2,r:1@256;row:1/2,col:4,r:2@256" --variants 0,2,4 --reps 5 --check > gpurun_out/p73/cfg4_n4.log 2>&1
tail -n 2 gpurun_out/p73/test.log; for n in 8 4; do grep -v Warn gpurun_out/p73/cfg4_n$n.log | head -7; grep -c OK gpurun_out/p73/cfg4_n$n.log; done
