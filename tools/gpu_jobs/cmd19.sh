python tools/experiments/ab_interleaved.py --config 2 --variants 5,12,1,13 --rounds 5 > gpurun_out/ab19_cfg2.log 2>&1
python tools/experiments/ab_interleaved.py --config 3 --variants 1,13,5,12 --rounds 5 > gpurun_out/ab19_cfg3.log 2>&1
python tools/experiments/ab_interleaved.py --config 5 --variants 9,14 --rounds 5 > gpurun_out/ab19_cfg5.log 2>&1
