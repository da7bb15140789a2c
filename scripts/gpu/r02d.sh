mkdir -p gpurun_out/r02d
timeout 300 python scripts/mb_argmax_bwd.py > gpurun_out/r02d/mb.log 2>&1
cat gpurun_out/r02d/mb.log
timeout 900 python -m pytest -x -q tests/test_concurrency_gpu.py tests/test_shim_cpp.py tests/test_bench_dist_gpu.py > gpurun_out/r02d/pytest.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/r02d/pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/r02d/cfg3_metrics.csv python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > gpurun_out/r02d/ncu_cfg3.log 2>&1
echo ncu_rc=$?
