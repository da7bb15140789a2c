# kbench + bench (device-resident value only) of the default lib and _var/<V> builds
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/var_bench.log; rm -f $o
for v in default ${VARS:-A B C}; do
  if [ $v = default ]; then L=""; else L=$PWD/paper_2007_06354_b200/_var/$v/lib/libgspmm_b200.so; fi
  echo "== $v" >> $o
  GSPMM_LIB_PATH=$L timeout 600 python scripts/kbench.py --cases ${KC:-rmat256,cfg2bwd,rmat100sym,rmat512h} >> $o 2>&1
  GSPMM_LIB_PATH=$L timeout 600 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'case':'bench','ms':round(d['ms_per_step'],4),'fwd':round(d['kernels_ms']['fwd'],4),'bwd':round(d['kernels_ms']['bwd'],4)}))" >> $o
done
