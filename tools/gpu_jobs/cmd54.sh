mkdir -p gpurun_out/p54
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/p54/launches.csv python tools/experiments/panel_launches.py > gpurun_out/p54/run.log 2>&1
tail -n 2 gpurun_out/p54/run.log
