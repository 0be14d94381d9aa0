python tools/experiments/ab_interleaved.py --config 2 --variants 5,12,13 --rounds 5 > gpurun_out/ab44_cfg2.log 2>&1
python tools/experiments/ab_interleaved.py --config 3 --variants 1,14,15 --rounds 5 > gpurun_out/ab44_cfg3.log 2>&1
