# r04f: max / min long rows in edge chunks by default: full GPU suite, cfg3 passes, kbench cases
O=gpurun_out/r04f
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python scripts/kb_cfg3.py - "" / split_edges=1 > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl | cut -c1-400
