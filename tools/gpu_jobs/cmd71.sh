# the driver's round-end commands at HEAD: reference arm, bench, GPU tests, smoke
mkdir -p gpurun_out/p71
( time timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/p71/ref.json 2> gpurun_out/p71/ref.err
( time timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/p71/bench.json 2> gpurun_out/p71/bench.err
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/p71/gt.log 2>&1; echo rc=$? >> gpurun_out/p71/gt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/p71/smoke.log 2>&1
head -c 400 gpurun_out/p71/ref.json; echo; tail -n 3 gpurun_out/p71/ref.err; head -c 300 gpurun_out/p71/bench.json; echo; tail -n 3 gpurun_out/p71/bench.err
tail -n 2 gpurun_out/p71/gt.log; tail -n 1 gpurun_out/p71/smoke.log
