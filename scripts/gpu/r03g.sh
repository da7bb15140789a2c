# r03g: larger long-row stages (more gathered bytes in flight per CTA): 48 KB x 3, 64 KB x 2
O=gpurun_out/r03g
mkdir -p $O
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in df12 df16nb2; do
  timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_ab/$v.so >> $O/kb.jsonl 2> $O/kb_$v.err
  cp paper_2007_06354_b200/_ab/$v.so paper_2007_06354_b200/_lib/libgspmm_b200.so
  timeout 600 python scripts/kbench.py --cases rmat256,rmat512h >> $O/kb2.jsonl 2>> $O/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
cat $O/kb.jsonl $O/kb2.jsonl
tail -3 $O/kb_df12.err
