# r02k: HEAD re-verified after the container was re-created: the whole GPU
# suite, smoke, the default bench (cfg3) with both arms, the launch list and
# per-kernel DRAM metrics of the cfg3 step, cfg2 bench.
mkdir -p gpurun_out/r02k
O=gpurun_out/r02k
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -5 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?"; tail -3 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.log
echo "bench cfg3 rc=$?"; cat $O/bench_cfg3.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_cfg3_reference.json 2> $O/bench_cfg3_reference.log
echo "bench ref rc=$?"; cat $O/bench_cfg3_reference.json
timeout 600 python bench.py --workload cfg2 --steps 10 --warmup 3 --skip-cpu > $O/bench_cfg2.json 2> $O/bench_cfg2.log
echo "bench cfg2 rc=$?"; cat $O/bench_cfg2.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum --clock-control none --csv --log-file $O/cfg3_metrics.csv python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > $O/ncu_cfg3.log 2>&1
echo ncu_rc=$?
timeout 600 python scripts/kb_cfg3.py - > $O/kb_cfg3.jsonl 2> $O/kb_cfg3.err
cat $O/kb_cfg3.jsonl
