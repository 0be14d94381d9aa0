mkdir -p gpurun_out/p64
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/p64/gt.log 2>&1; echo rc=$? >> gpurun_out/p64/gt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/p64/smoke.log 2>&1
tail -n 3 gpurun_out/p64/gt.log; tail -n 2 gpurun_out/p64/smoke.log
