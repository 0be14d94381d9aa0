python -m pytest tests/test_gpu_scale.py tests/test_gpu_baseline_shapes.py -x -q -p no:cacheprovider -k "config2 or config3 or config5 or exact_rows or cold_column" > gpurun_out/gt32.log 2>&1; echo rc=$? >> gpurun_out/gt32.log
run() { SGAP_LIB=$2 python tools/experiments/ab_interleaved.py --config $3 --variants $4 --rounds 4 2>/dev/null | grep median | sed "s/^/$1 cfg$3 /"; }
for rep in 1 2; do
  run new paper_2209_02882_b200/libsgap.so 2 5,1 >> gpurun_out/ab32.log
  run old tools/experiments/alt/libsgap.so 2 5,1 >> gpurun_out/ab32.log
  run new paper_2209_02882_b200/libsgap.so 3 1 >> gpurun_out/ab32.log
  run old tools/experiments/alt/libsgap.so 3 1 >> gpurun_out/ab32.log
  run new paper_2209_02882_b200/libsgap.so 5 9 >> gpurun_out/ab32.log
  run old tools/experiments/alt/libsgap.so 5 9 >> gpurun_out/ab32.log
done
