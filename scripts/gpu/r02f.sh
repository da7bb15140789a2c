mkdir -p gpurun_out/r02f
timeout 600 python -m pytest -x -q tests/test_parity_gpu.py -k "second_reduction or long_row or granularity or register_path" > gpurun_out/r02f/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02f/pytest.log
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in v0 v4 v5; do
  timeout 300 python scripts/kb_cfg3.py paper_2007_06354_b200/_var/$v.so >> gpurun_out/r02f/kb.jsonl 2> gpurun_out/r02f/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
cat gpurun_out/r02f/kb.jsonl
