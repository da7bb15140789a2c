# r04h: argmax fold with FFMA / IMAD conditional copies (FMA pipes) against FSEL / SEL (ALU pipe)
O=gpurun_out/r04h
mkdir -p $O
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_ab/fma0.so > $O/kb.jsonl 2> $O/kb_fma0.err
timeout 600 python scripts/kb_cfg3.py /tmp/intree.so >> $O/kb.jsonl 2> $O/kb_fma1.err
timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_ab/fma0.so >> $O/kb.jsonl 2>> $O/kb_fma0.err
timeout 600 python scripts/kb_cfg3.py /tmp/intree.so >> $O/kb.jsonl 2>> $O/kb_fma1.err
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
cut -c1-300 $O/kb.jsonl
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.log
