# r02m: the straight-line long-row fold (LG_FOLD) and column-major narrow
# stages (LG_TR): parity, then A/B against the previous fold on the cfg3 passes.
mkdir -p gpurun_out/r02m
O=gpurun_out/r02m
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_io_gpu.py tests/test_concurrency_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 300 python scripts/sanitize_case.py 2>&1 | tail -1
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in f0 f1; do
  timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_ab/$v.so >> $O/kb.jsonl 2> $O/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
timeout 600 python scripts/kb_cfg3.py - >> $O/kb.jsonl 2> $O/kb_intree.err
cat $O/kb.jsonl
timeout 1200 python -m pytest -x -q tests/test_scale_gpu.py > $O/pytest_scale.log 2>&1
echo "scale rc=$?"; tail -5 $O/pytest_scale.log
