mkdir -p gpurun_out/r02h
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in v0 p0 p1; do
  timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_var/$v.so long_serial=1 / "" / long_ctas=74 >> gpurun_out/r02h/kb.jsonl 2> gpurun_out/r02h/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
cat gpurun_out/r02h/kb.jsonl
