# cfg5/long-row knob sweep (development aid)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/cfg5_ab.log; rm -f $out
C=${C:-cfg5mean}
echo "== trace" >> $out; timeout 300 python scripts/trace_case.py $C >> $out 2>&1
for kv in "X=0" "GSPMM_LONG_EDGES=30000" "GSPMM_LONG_EDGES=16384" "GSPMM_XL_EDGES=100000" \
          "GSPMM_LONG_CTAS=148" "GSPMM_LONG_TMA=1"; do
  echo "== $kv" >> $out
  env $kv timeout 300 python scripts/kbench.py --cases $C >> $out 2>&1
done
