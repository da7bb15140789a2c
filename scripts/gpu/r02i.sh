mkdir -p gpurun_out/r02i
timeout 900 python scripts/kb_cfg3.py - long_serial=1 / long_serial=1 unit_cols=32 / long_serial=1 unit_cols=100 / long_serial=1 long_threshold=65536 / long_serial=1 long_threshold=32768 / long_serial=1 long_threshold=8192 > gpurun_out/r02i/kb.jsonl 2> gpurun_out/r02i/kb.err
cat gpurun_out/r02i/kb.jsonl
timeout 900 ncu --set full --import-source on -k regex:k_long_rg -c 2 -o gpurun_out/r02i/long python scripts/kb_cfg3.py - long_serial=1 > gpurun_out/r02i/ncu.log 2>&1
echo ncu rc=$?
