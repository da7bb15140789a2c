# r03b: segment geometry for 129..256-column units (cfg2 / cfg4 shapes)
O=gpurun_out/r03b
mkdir -p $O
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in v2b5 v2b6 v4b4 v1b6; do
  cp paper_2007_06354_b200/_ab/$v.so paper_2007_06354_b200/_lib/libgspmm_b200.so
  echo "{\"variant\": \"$v\"}" >> $O/kb.jsonl
  timeout 600 python scripts/kbench.py --cases rmat256,cfg2bwd,rmat512h,er256 >> $O/kb.jsonl 2>> $O/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
cat $O/kb.jsonl
