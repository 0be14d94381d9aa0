python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gt17.log 2>&1; echo rc=$? >> gpurun_out/gt17.log
timeout 2400 python tools/paper_claims.py --matrices cfg2,cfg3,cfg4 --n 4,16,64,128 --out gpurun_out/claims_cfg234_v2.json > gpurun_out/claims17.log 2>&1
