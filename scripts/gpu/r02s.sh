# r02s: lean producer with one / two stages of gathers in flight, KQ 6 / 7
mkdir -p gpurun_out/r02s
O=gpurun_out/r02s
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in l1k7 l2k6 l2k7; do
  timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_ab/$v.so >> $O/kb.jsonl 2> $O/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
cat $O/kb.jsonl
