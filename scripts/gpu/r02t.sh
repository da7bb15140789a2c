# r02t: item-spread producer + block fold / tree argmax / compile-time narrow strides
mkdir -p gpurun_out/r02t
O=gpurun_out/r02t
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_concurrency_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python scripts/sanitize_case.py 2>&1 | tail -1
timeout 600 python scripts/kb_cfg3.py - > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl
