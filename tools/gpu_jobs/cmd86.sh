# config-4 N sweep re-run with the shifted-block walk in the candidate set (kbench --all)
mkdir -p gpurun_out/p86
for n in 16 32 64 128 256 512; do
  timeout 1200 python tools/kbench.py --config 4 --n $n --all --reps 3 --out gpurun_out/p86/sweep_cfg4_n$n.json > gpurun_out/p86/sweep_cfg4_n$n.log 2>&1
done
python tools/sweep_table.py gpurun_out/p86/sweep_cfg4_n*.json
