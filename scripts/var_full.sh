# variants: kbench + long-row unit traces (development aid)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/var_full.log; rm -f $out
for v in ${VARS:-A B}; do
  echo "== variant $v" >> $out
  export GSPMM_LIB_PATH=$PWD/paper_2007_06354_b200/_var/$v/lib/libgspmm_b200.so
  timeout 600 python scripts/kbench.py --cases ${K:-rmat256,rmat512h,rmat100sym,cfg3max} >> $out 2>&1
  timeout 300 python scripts/trace_case.py ${TC:-rmat256} 2>&1 | grep -E "rows" >> $out
done
