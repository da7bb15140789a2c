# A/B of the long-row kernels (development aid)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/async_ab.log; rm -f $out
for la in ${PYLA:-2}; do
  GSPMM_LONG_ASYNC=$la timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not scale" > gpurun_out/async_pytest_$la.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/async_pytest_$la.log
done
K=${K:-cfg5mean,rmat256,star256,rmat100sym,rmat512h,cfg3max}
for kv in ${KVS:-X=0 GSPMM_LONG_ASYNC=1 GSPMM_LONG_ASYNC=2}; do
  echo "== $kv" >> $out
  env $kv timeout 600 python scripts/kbench.py --cases $K >> $out 2>&1
  env $kv timeout 300 python scripts/trace_case.py ${TC:-rmat256} 2>&1 | grep "rows" >> $out
done
