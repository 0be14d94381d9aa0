python tools/experiments/ab_interleaved.py --config 3 --n 256 --point nnz:512,col:4,r:1 --variants 1,5,9 --hints --rounds 4 > gpurun_out/ab23_cfg3_n256.log 2>&1
python tools/experiments/ab_interleaved.py --config 4 --n 512 --point nnz:128,col:4,r:1 --variants 1,5,9 --hints --rounds 4 > gpurun_out/ab23_cfg4_n512.log 2>&1
python tools/experiments/ab_interleaved.py --config 2 --point nnz:512,col:4,r:1 --variants 5,9 --hints --rounds 4 > gpurun_out/ab23_cfg2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke23.log 2>&1
