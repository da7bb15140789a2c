# r04z: final evidence of round 2 at HEAD: the whole GPU suite, smoke, the default
# bench (cfg3) with both arms, launch list + per-kernel DRAM / L2 metrics of
# the cfg3 step, --set full captures of the two dominant kernels, the other
# workloads' bench lines, every kbench case, the long-row unit timeline.
O=gpurun_out/r04z
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 300 python scripts/sanitize_case.py > $O/sanitize_case.log 2>&1; tail -1 $O/sanitize_case.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.log
echo "bench cfg3 rc=$?"; cat $O/bench_cfg3.json
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_cfg3_reference.json 2> $O/bench_cfg3_reference.log
echo "bench ref rc=$?"; cat $O/bench_cfg3_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum --clock-control none --csv --log-file $O/cfg3_metrics.csv python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > $O/ncu_cfg3.log 2>&1
echo ncu_metrics_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather --launch-skip 6 -c 2 -o $O/gather python bench.py --steps 1 --warmup 3 --skip-e2e --skip-cpu > $O/ncu_full.log 2>&1
echo ncu_full_rc=$?
for w in cfg2 cfg1 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --skip-cpu > $O/bench_$w.json 2> $O/bench_$w.log
  echo "bench $w rc=$?"; cut -c1-400 $O/bench_$w.json
done
timeout 1500 python scripts/kbench.py --cases er128,er256,rmat256,rmatcap256,rmat100sym,cfg3max,rmat512h,cfg5mean,cfg2dot,cfg4dot,cfg4softmax,cfg2bwd,cfg3meanbwd,cfg3maxbwd,cfg4bwdx,cfg5meanbwd,cfg4softmaxbwd > $O/kbench.jsonl 2> $O/kbench.err
cat $O/kbench.jsonl
timeout 600 python scripts/kb_cfg3.py - > $O/kb_cfg3.jsonl 2> $O/kb_cfg3.err
cat $O/kb_cfg3.jsonl

timeout 900 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-e2e --split-edges 512 > $O/bench_cfg3_split512.json 2> $O/bench_cfg3_split512.log
echo "bench split rc=$?"; cut -c1-300 $O/bench_cfg3_split512.json
