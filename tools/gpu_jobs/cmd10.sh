# both bench arms as the driver runs them (N=1), plus the gpu tests
( time python bench.py --impl reference > gpurun_out/ref10.json 2> gpurun_out/ref10.err ) 2> gpurun_out/ref10.time
( time python bench.py > gpurun_out/b10.json 2> gpurun_out/b10.err ) 2> gpurun_out/b10.time
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt10.log 2>&1; echo rc=$? >> gpurun_out/gt10.log
