# r02y: plan level 8192 added (cfg4: 8.23 -> 7.08 ms with rows above 8192 as long rows)
O=gpurun_out/r02y
mkdir -p $O
timeout 900 python scripts/kbench.py --cases rmat256,cfg2bwd,rmat512h,cfg4bwdx,cfg5mean,er256 > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl
timeout 600 python scripts/kb_cfg3.py - > $O/kb_cfg3.jsonl 2> $O/kb_cfg3.err
cat $O/kb_cfg3.jsonl
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.log
