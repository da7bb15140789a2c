# kbench of the default lib and the _var/<V> builds, interleaved (A/B on one box)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/var_kb.log; rm -f $o
C=${KC:-er128,rmat256,rmat512h}
for rep in 1 2; do for v in default ${VARS:-A B}; do
  echo "== $v" >> $o
  if [ $v = default ]; then timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1
  else GSPMM_LIB_PATH=$PWD/paper_2007_06354_b200/_var/$v/lib/libgspmm_b200.so timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1; fi
done; done
