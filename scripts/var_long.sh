# long-row ring-geometry variants (development aid)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/var_long.log; rm -f $out
K=${K:-cfg5mean,rmat256,rmat100sym,rmat512h,cfg3max}
for v in ${VARS:-A B C D}; do
  echo "== variant $v" >> $out
  export GSPMM_LIB_PATH=$PWD/paper_2007_06354_b200/_var/$v/lib/libgspmm_b200.so GSPMM_LONG_ASYNC=${LA:-1}
  timeout 600 python scripts/kbench.py --cases $K >> $out 2>&1
  timeout 300 python scripts/trace_case.py rmat256 2>&1 | grep "rows" >> $out
done
