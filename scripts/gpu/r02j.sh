mkdir -p gpurun_out/r02j
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in w0 w1 w2; do
  timeout 600 python scripts/kb_cfg3.py paper_2007_06354_b200/_var/$v.so >> gpurun_out/r02j/kb.jsonl 2> gpurun_out/r02j/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
cat gpurun_out/r02j/kb.jsonl
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather --launch-skip 26 -c 1 -o gpurun_out/r02j/dual_gather python scripts/kb_cfg3.py - > gpurun_out/r02j/ncu.log 2>&1
echo ncu rc=$?
