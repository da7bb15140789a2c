# r04e: split_edges parity test after the tolerance correction
O=gpurun_out/r04e
mkdir -p $O
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "split_by_edges" > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -15 $O/pytest.log
