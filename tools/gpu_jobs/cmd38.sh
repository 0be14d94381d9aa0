python tools/experiments/ab_interleaved.py --config 5 --variants 9,18,1,17 --rounds 5 > gpurun_out/ab38_cfg5.log 2>&1
python tools/experiments/ab_interleaved.py --config 2 --variants 5,1,17 --rounds 5 > gpurun_out/ab38_cfg2.log 2>&1
python tools/experiments/ab_interleaved.py --config 3 --variants 1,17 --rounds 5 --hints > gpurun_out/ab38_cfg3.log 2>&1
