# r04i: HEAD after the FFMA value copy in the argmax fold: GPU suite, smoke, the default bench
# line, launch list + DRAM metrics, --set full of the two segment instances, cfg3 passes
O=gpurun_out/r04i
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 300 python scripts/sanitize_case.py > $O/sanitize_case.log 2>&1; tail -1 $O/sanitize_case.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.log
echo "bench cfg3 rc=$?"; cut -c1-500 $O/bench_cfg3.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum --clock-control none --csv --log-file $O/cfg3_metrics.csv python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > $O/ncu_cfg3.log 2>&1
echo ncu_metrics_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather --launch-skip 6 -c 2 -o $O/gather python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > $O/ncu_full.log 2>&1
echo ncu_full_rc=$?
timeout 600 python scripts/kb_cfg3.py - > $O/kb_cfg3.jsonl 2> $O/kb_cfg3.err
cat $O/kb_cfg3.jsonl
timeout 900 python scripts/kbench.py --cases cfg3max,rmat100sym,rmat256,rmat512h > $O/kbench.jsonl 2> $O/kbench.err
cut -c1-250 $O/kbench.jsonl
