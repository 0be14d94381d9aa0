timeout 1800 python tools/scaling_projection.py --strong --unpermuted --worlds 1,2,4,8 --variant 9 --out gpurun_out/r02_scaling_projection_unpermuted_nnz.json > gpurun_out/scal30a.log 2>&1
timeout 1800 python tools/scaling_projection.py --strong --unpermuted --balance bytes --worlds 1,2,4,8 --variant 9 --out gpurun_out/r02_scaling_projection_unpermuted_bytes.json > gpurun_out/scal30b.log 2>&1
