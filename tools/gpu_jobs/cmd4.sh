for n in 16 32 64 128 256 512; do
  timeout 900 python tools/kbench.py --config 4 --n $n --all --reps 3 --out gpurun_out/sweep_cfg4_n$n.json > gpurun_out/sweep_cfg4_n$n.log 2>&1
done
for n in 64 256; do
  timeout 900 python tools/kbench.py --config 3 --n $n --all --reps 3 --out gpurun_out/sweep_cfg3_n$n.json > gpurun_out/sweep_cfg3_n$n.log 2>&1
done
timeout 900 python tools/kbench.py --config 2 --n 128 --all --reps 3 --out gpurun_out/sweep_cfg2_n128.json > gpurun_out/sweep_cfg2_n128.log 2>&1
timeout 2400 python tools/paper_claims.py --matrices cfg2,cfg3,cfg4 --n 4,16,64,128 --out gpurun_out/claims_cfg234.json > gpurun_out/claims.log 2>&1
