# r04m: long-row units handed out by measured unit time (LPT on the fitted model)
O=gpurun_out/r04m
mkdir -p $O
timeout 600 python scripts/kb_cfg3.py - "" / "" > $O/kb.jsonl 2> $O/kb.err
cut -c1-200 $O/kb.jsonl
timeout 900 python scripts/kbench.py --cases rmat256,rmat512h,cfg2bwd > $O/kbench.jsonl 2> $O/kbench.err
cut -c1-150 $O/kbench.jsonl
