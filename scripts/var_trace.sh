# per-variant long-row unit traces (development aid)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/var_trace.log; rm -f $out
for v in ${VARS:-A B C}; do
  echo "== variant $v" >> $out
  GSPMM_LIB_PATH=$PWD/paper_2007_06354_b200/_var/$v/lib/libgspmm_b200.so timeout 300 python scripts/trace_case.py ${TC:-rmat256} 2>&1 | grep -E "rows|mode" >> $out
done
