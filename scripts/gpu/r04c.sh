# r04c: long rows split by edges (plan split_edges): parity test, then cfg3 / cfg2 / cfg4 timings
O=gpurun_out/r04c
mkdir -p $O
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "split_by_edges" > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -15 $O/pytest.log
timeout 900 python scripts/kb_cfg3.py - "" / split_edges=512 / split_edges=256 / split_edges=1024 / split_edges=512 long_threshold=4096 / split_edges=512 long_threshold=8192 / split_edges=1024 long_threshold=2048 > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl | cut -c1-400
timeout 900 python scripts/kbench.py --cases rmat256,cfg2bwd,rmat512h,cfg4bwdx --plans " / split_edges=512 / split_edges=256 / split_edges=512 long_threshold=2048 / split_edges=512 long_threshold=1024" > $O/kb2.jsonl 2> $O/kb2.err
cut -c1-300 $O/kb2.jsonl
