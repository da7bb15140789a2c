# r04a: the long-row / segment kernel pair as a programmatic dependent launch (default)
# against strictly serial launches (plan kernel=2): cfg3 passes, cfg2 / cfg4 shapes, parity
O=gpurun_out/r04a
mkdir -p $O
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_concurrency_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 900 python scripts/kb_cfg3.py - "" / kernel=2 / "" / kernel=2 > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl | cut -c1-400
timeout 900 python scripts/kbench.py --cases rmat256,cfg2bwd,rmat512h,cfg4bwdx --plans " / kernel=2" > $O/kb2.jsonl 2> $O/kb2.err
cut -c1-300 $O/kb2.jsonl
