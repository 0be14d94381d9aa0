python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt20.log 2>&1; echo rc=$? >> gpurun_out/gt20.log
python tools/experiments/ab_interleaved.py --config 2 --variants 5,1 --rounds 5 > gpurun_out/ab20_cfg2.log 2>&1
python tools/experiments/ab_interleaved.py --config 3 --variants 1,5 --rounds 5 > gpurun_out/ab20_cfg3.log 2>&1
python tools/experiments/ab_interleaved.py --config 5 --variants 9,1,5 --rounds 5 > gpurun_out/ab20_cfg5.log 2>&1
