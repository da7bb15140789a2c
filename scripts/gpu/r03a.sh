# r03a: two segment geometries for <= 128 columns chosen by the gathered table size
O=gpurun_out/r03a
mkdir -p $O
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_concurrency_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python scripts/sanitize_case.py 2>&1 | tail -1
timeout 600 python scripts/kb_cfg3.py - > $O/kb_cfg3.jsonl 2> $O/kb_cfg3.err
cat $O/kb_cfg3.jsonl
timeout 900 python scripts/kbench.py --cases er128,rmat256,rmat512h,cfg5mean > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl
timeout 1500 python -m pytest -x -q tests/test_scale_gpu.py > $O/pytest_scale.log 2>&1
echo "scale rc=$?"; tail -3 $O/pytest_scale.log
