# r02z: segment kernel geometry (edges per batch x blocks per SM) for the <= 128-column instances,
# DUAL / ARG included, on the cfg3 passes and the cfg1 shape
O=gpurun_out/r02z
mkdir -p $O
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in u4b6 u2b6 u2b8 u4b5; do
  timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_ab/$v.so >> $O/kb.jsonl 2> $O/kb_$v.err
  timeout 300 python scripts/kbench.py --cases er128 >> $O/kb_er128.jsonl 2>> $O/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
timeout 300 python scripts/kbench.py --cases er128 >> $O/kb_er128.jsonl 2>> $O/kb_intree.err
cat $O/kb.jsonl $O/kb_er128.jsonl
