# r03l: the new large-table geometry test
mkdir -p gpurun_out/r03l
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "large_table or zero_width or ties_zeros" > gpurun_out/r03l/pytest.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/r03l/pytest.log
