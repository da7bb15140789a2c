# edge-destined dot variants: parity subset + kbench (default, _var builds, old k_dot_edges4)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/dot_ab.log; rm -f $o
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_dot.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dot.log
C=${KC:-cfg2dot,cfg4dot}
for v in default ${VARS:-A B C} old; do
  echo "== $v" >> $o
  if [ $v = default ]; then timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1
  elif [ $v = old ]; then GSPMM_DOT_EDGES=4 timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1
  else GSPMM_LIB_PATH=$PWD/paper_2007_06354_b200/_var/$v/lib/libgspmm_b200.so timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1; fi
done
