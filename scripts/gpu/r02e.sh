# long-row kernel variants (ids ahead, stage size, data stages) on the cfg3 passes
mkdir -p gpurun_out/r02e
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
for v in v0 v1 v2 v3; do
  timeout 300 python scripts/kb_cfg3.py paper_2007_06354_b200/_var/$v.so >> gpurun_out/r02e/kb.jsonl 2> gpurun_out/r02e/kb_$v.err
done
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
cat gpurun_out/r02e/kb.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/r02e/v0_metrics.csv python scripts/kb_cfg3.py paper_2007_06354_b200/_var/v0.so > /dev/null 2>&1
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
echo done
