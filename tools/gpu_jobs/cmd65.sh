mkdir -p gpurun_out/p65
timeout 900 python tools/experiments/stencil_panel_probe.py --n 512 > gpurun_out/p65/n512.log 2>&1
timeout 900 python tools/experiments/stencil_panel_probe.py --n 256 --full "nnz:128,col:4,r:1@1024/1;row:32,col:4,r:1@1024/0" > gpurun_out/p65/n256.log 2>&1
tail -n 5 gpurun_out/p65/*.log
