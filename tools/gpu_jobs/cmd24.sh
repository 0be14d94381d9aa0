python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt24.log 2>&1; echo rc=$? >> gpurun_out/gt24.log
run() { # label lib config n points variants
  SGAP_LIB=$2 python tools/kbench.py --config $3 --n $4 --points "$5" --variants $6 --reps 7 2>/dev/null | grep " ms " | grep -v cuSPARSE | sed "s/^/$1 cfg$3 n$4 /"
}
for rep in 1 2; do
  run new paper_2209_02882_b200/libsgap.so 3 256 "nnz:512,col:4,r:1@1024" 1,5 >> gpurun_out/ab24.log
  run old tools/experiments/alt/libsgap.so 3 256 "nnz:512,col:4,r:1@1024" 1,5 >> gpurun_out/ab24.log
  run new paper_2209_02882_b200/libsgap.so 4 512 "nnz:128,col:4,r:1@1024" 1,5 >> gpurun_out/ab24.log
  run old tools/experiments/alt/libsgap.so 4 512 "nnz:128,col:4,r:1@1024" 1,5 >> gpurun_out/ab24.log
  run new paper_2209_02882_b200/libsgap.so 4 256 "nnz:128,col:4,r:1@1024" 1,5 >> gpurun_out/ab24.log
  run old tools/experiments/alt/libsgap.so 4 256 "nnz:128,col:4,r:1@1024" 1,5 >> gpurun_out/ab24.log
done
