# r02p: per-unit timeline of the long-row kernel (LG_TRACE build) on cfg3
mkdir -p gpurun_out/r02p
O=gpurun_out/r02p
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
timeout 600 python scripts/trace_long.py paper_2007_06354_b200/_ab/${TV:-t1}.so mean > $O/trace_mean.txt 2> $O/trace_mean.err
timeout 600 python scripts/trace_long.py paper_2007_06354_b200/_ab/${TV:-t1}.so dual > $O/trace_dual.txt 2> $O/trace_dual.err
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
python scripts/trace_long_summary.py $O/trace_mean.txt
python scripts/trace_long_summary.py $O/trace_dual.txt
