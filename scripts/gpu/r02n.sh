# r02n: producer depth / stage size / column-major variants of the long-row kernel on cfg3
mkdir -p gpurun_out/r02n
O=gpurun_out/r02n
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in g1 g2 g3 g4; do
  timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_ab/$v.so >> $O/kb.jsonl 2> $O/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
cat $O/kb.jsonl
