# r04l: plan level for the exact edge-chunk path of max / min (read the max+argmax column only)
O=gpurun_out/r04l
mkdir -p $O
timeout 900 python scripts/kb_cfg3.py - "" / long_threshold=8192 / long_threshold=4096 / long_threshold=2048 / long_threshold=1024 / long_threshold=4096 split_edges=256 / long_threshold=4096 split_edges=1024 > $O/kb.jsonl 2> $O/kb.err
cut -c1-200 $O/kb.jsonl
