mkdir -p gpurun_out/p57
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/p57/gt.log 2>&1; echo rc=$? >> gpurun_out/p57/gt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/p57/smoke.log 2>&1
timeout 600 python tools/experiments/ab_interleaved.py --config 3 --n 256 --variants 1,10 --rounds 5 > gpurun_out/p57/ab_cfg3_n256.log 2>&1
tail -n 3 gpurun_out/p57/gt.log; tail -n 2 gpurun_out/p57/smoke.log; tail -n 3 gpurun_out/p57/ab_cfg3_n256.log
