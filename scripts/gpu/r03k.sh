# r03k: long-row kernel capped at 96 / 80 registers so a segment block can share its SM;
# serial order vs concurrent on all 148 SMs (plan long_ctas=148)
O=gpurun_out/r03k
mkdir -p $O
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in mr96 mr80; do
  timeout 900 python scripts/kb_cfg3.py paper_2007_06354_b200/_ab/$v.so "" / long_ctas=148 / long_ctas=100 >> $O/kb.jsonl 2> $O/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
timeout 600 python scripts/kb_cfg3.py - long_ctas=148 >> $O/kb.jsonl 2> $O/kb_intree.err
cat $O/kb.jsonl
