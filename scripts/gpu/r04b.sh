# r04b: cfg2 shape, long-row threshold below the 4096 level (segment rows as one warp's sequential work)
O=gpurun_out/r04b
mkdir -p $O
timeout 900 python scripts/kbench.py --cases rmat256,cfg2bwd --plans " / long_threshold=3072 / long_threshold=2048 / long_threshold=1536 / long_threshold=1024 / long_threshold=2048 seg_cost=128 / long_threshold=2048 seg_cost=512" > $O/kb.jsonl 2> $O/kb.err
cut -c1-300 $O/kb.jsonl
timeout 900 python scripts/kbench.py --cases rmat512h --plans " / long_threshold=6144 / long_threshold=4096 / long_threshold=12288" > $O/kb4.jsonl 2> $O/kb4.err
cut -c1-300 $O/kb4.jsonl
