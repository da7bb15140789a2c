# per-variant long-row unit traces + kbench (development aid)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/var_trace.log; rm -f $out
for v in default ${VARS:-A B C}; do
  echo "== variant $v" >> $out
  if [ $v = default ]; then L=""; else L=$PWD/paper_2007_06354_b200/_var/$v/lib/libgspmm_b200.so; fi
  for c in ${TC:-rmat256}; do
    GSPMM_LIB_PATH=$L timeout 300 python scripts/trace_case.py $c 2>&1 | grep -E "rows|mode" >> $out
    GSPMM_LIB_PATH=$L timeout 300 python scripts/kbench.py --cases $c 2>&1 | grep case >> $out
  done
done
