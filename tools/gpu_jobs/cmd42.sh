python tools/experiments/ab_interleaved.py --config 2 --variants 5,10 --rounds 6 --hints > gpurun_out/ab42_cfg2.log 2>&1
python tools/experiments/ab_interleaved.py --config 5 --variants 9,10 --rounds 4 > gpurun_out/ab42_cfg5.log 2>&1
python tools/experiments/ab_interleaved.py --config 3 --n 256 --variants 1,9,10 --rounds 4 --hints > gpurun_out/ab42_cfg3.log 2>&1
