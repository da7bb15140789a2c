# r03e: after the systolic edge-dot experiment was reverted: the whole GPU
# suite again, the cfg4 bench line and the dot kbench cases
O=gpurun_out/r03e
mkdir -p $O
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py --workload cfg4 --steps 10 --warmup 3 --skip-cpu > $O/bench_cfg4.json 2> $O/bench_cfg4.log
echo "bench cfg4 rc=$?"; cut -c1-600 $O/bench_cfg4.json
timeout 900 python scripts/kbench.py --cases cfg2dot,cfg4dot > $O/kbench_dot.jsonl 2> $O/kbench_dot.err
cat $O/kbench_dot.jsonl
