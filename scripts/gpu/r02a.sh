set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --workload cfg3 --steps 5 --warmup 3 --skip-e2e > gpurun_out/r02a/bench_cfg3.json 2> gpurun_out/r02a/bench_cfg3.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r02a/cfg3_metrics.csv python bench.py --workload cfg3 --steps 1 --warmup 3 --skip-e2e > gpurun_out/r02a/ncu_cfg3.log 2>&1
echo ncu_rc=$?
