# r02x: cfg4 forward under threshold x concurrency plan variants
O=gpurun_out/r02x
mkdir -p $O
timeout 900 python scripts/kbench.py --cases rmat512h --plans "long_threshold=16384 long_ctas=16 / long_threshold=16384 long_ctas=32 / long_threshold=16384 long_ctas=74 / long_threshold=32768 / long_threshold=32768 long_ctas=16 / long_threshold=32768 long_ctas=32 / long_threshold=8192 / long_threshold=8192 long_ctas=32 / long_threshold=4096 / long_threshold=2048 / seg_cost=512 long_threshold=16384" > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl
