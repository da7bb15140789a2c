# r02u: long-row units concurrent with the segment kernel (plan option long_ctas) after the r02t kernel
mkdir -p gpurun_out/r02u
timeout 900 python scripts/kb_cfg3.py - "" / long_ctas=16 / long_ctas=32 / long_ctas=48 / long_threshold=32768 / long_threshold=65536 > gpurun_out/r02u/kb.jsonl 2> gpurun_out/r02u/kb.err
cat gpurun_out/r02u/kb.jsonl
