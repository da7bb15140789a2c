# r02q: rewritten long-row kernel (warp-per-edges producer, compile-time-stride
# narrow consumer): parity, cfg3 passes, unit trace
mkdir -p gpurun_out/r02q
O=gpurun_out/r02q
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_concurrency_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 300 python scripts/sanitize_case.py 2>&1 | tail -1
timeout 600 python scripts/kb_cfg3.py - > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
timeout 600 python scripts/trace_long.py paper_2007_06354_b200/_ab/t1.so mean > $O/trace_mean.txt 2> $O/trace_mean.err
timeout 600 python scripts/trace_long.py paper_2007_06354_b200/_ab/t1.so dual > $O/trace_dual.txt 2> $O/trace_dual.err
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
python scripts/trace_long_summary.py $O/trace_mean.txt
python scripts/trace_long_summary.py $O/trace_dual.txt
