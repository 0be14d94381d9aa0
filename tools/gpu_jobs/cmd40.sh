python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt40.log 2>&1; echo rc=$? >> gpurun_out/gt40.log
python bench.py > gpurun_out/b40.json 2> gpurun_out/b40.err
