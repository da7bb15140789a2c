# r02v: round-end evidence at HEAD: the whole GPU suite, smoke, the default
# bench (cfg3) with both arms, launch list + per-kernel DRAM / L2 metrics of
# the cfg3 step, one --set full capture of the dominant kernel, cfg2 / cfg1 /
# cfg4 / cfg5 bench lines.
O=gpurun_out/r02v
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.log
echo "bench cfg3 rc=$?"; cat $O/bench_cfg3.json
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_cfg3_reference.json 2> $O/bench_cfg3_reference.log
echo "bench ref rc=$?"; cat $O/bench_cfg3_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum --clock-control none --csv --log-file $O/cfg3_metrics.csv python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > $O/ncu_cfg3.log 2>&1
echo ncu_metrics_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather --launch-skip 6 -c 1 -o $O/gather_dual python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > $O/ncu_full.log 2>&1
echo ncu_full_rc=$?
for w in cfg2 cfg1 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --skip-cpu > $O/bench_$w.json 2> $O/bench_$w.log
  echo "bench $w rc=$?"; cut -c1-700 $O/bench_$w.json
done
