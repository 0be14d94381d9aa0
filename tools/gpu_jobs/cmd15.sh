python -m pytest tests/test_gpu_scale.py -x -q -p no:cacheprovider -k "cold_column or exact_rows or long_chunk" > gpurun_out/gt15.log 2>&1; echo rc=$? >> gpurun_out/gt15.log
python tools/experiments/ab_interleaved.py --config 2 --variants 5,1,10 --rounds 5 > gpurun_out/ab15_cfg2.log 2>&1
python tools/experiments/ab_interleaved.py --config 3 --variants 1,5,10 --rounds 5 > gpurun_out/ab15_cfg3.log 2>&1
python tools/experiments/ab_interleaved.py --config 5 --variants 9,11,1,10 --rounds 5 > gpurun_out/ab15_cfg5.log 2>&1
