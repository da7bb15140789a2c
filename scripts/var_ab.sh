cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/var_ab.log
for v in ${VARS:-A B}; do
  echo "== variant $v" >> gpurun_out/var_ab.log
  GSPMM_LIB_PATH=$PWD/paper_2007_06354_b200/_var/$v/lib/libgspmm_b200.so timeout 400 python scripts/kbench.py --cases er128,er256,rmat256,rmat100sym >> gpurun_out/var_ab.log 2>&1
done
