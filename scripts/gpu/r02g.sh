mkdir -p gpurun_out/r02g
timeout 600 python -m pytest -x -q tests/test_parity_gpu.py -k "second_reduction or long_row or granularity or register_path" > gpurun_out/r02g/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02g/pytest.log
timeout 900 python scripts/kb_cfg3.py - "" / long_serial=1 / long_ctas=16 / long_ctas=32 / long_ctas=48 / long_ctas=74 / long_threshold=4096 / long_threshold=4096 long_serial=1 > gpurun_out/r02g/kb.jsonl 2> gpurun_out/r02g/kb.err
cat gpurun_out/r02g/kb.jsonl
