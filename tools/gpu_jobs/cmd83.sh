# pitch-ordered traversal of the shifted-block walk (experiment)
mkdir -p gpurun_out/p83
timeout 900 python tools/experiments/pitch_probe.py 128 > gpurun_out/p83/pitch_n128.log 2>&1
timeout 900 python tools/experiments/pitch_probe.py 256 > gpurun_out/p83/pitch_n256.log 2>&1
grep -v Warn gpurun_out/p83/pitch_n128.log gpurun_out/p83/pitch_n256.log | grep -v "bitwise True"
