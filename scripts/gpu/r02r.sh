# r02r: producer pacing of narrow long-row units (LG_PACE 0 / 20 / 40 / 70 % of the chain time)
mkdir -p gpurun_out/r02r
O=gpurun_out/r02r
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in p0 p20 p70; do
  timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_ab/$v.so >> $O/kb.jsonl 2> $O/kb_$v.err
done
timeout 600 python scripts/trace_long.py paper_2007_06354_b200/_ab/p40.so mean > $O/trace_mean.txt 2> $O/trace_mean.err
timeout 600 python scripts/trace_long.py paper_2007_06354_b200/_ab/p40.so dual > $O/trace_dual.txt 2> $O/trace_dual.err
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
timeout 600 python scripts/kb_cfg3.py - >> $O/kb.jsonl 2> $O/kb_intree.err
cat $O/kb.jsonl
python scripts/trace_long_summary.py $O/trace_mean.txt
python scripts/trace_long_summary.py $O/trace_dual.txt
