# r03d: systolic edge-dot kernel (k_dot_sys): parity, then the dot cases
O=gpurun_out/r03d
mkdir -p $O
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_autograd_gpu.py tests/test_shim_cpp.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 300 python scripts/sanitize_case.py 2>&1 | tail -1
timeout 900 python scripts/kbench.py --cases cfg2dot,cfg4dot > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl
