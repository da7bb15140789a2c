# env-knob sweep over kbench cases (development aid)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; out=gpurun_out/knob_ab.log; rm -f $out
K=${K:-rmat256,rmat100sym,rmat512h,cfg3max,star256}
for kv in ${KVS:-X=0}; do
  echo "== $kv" >> $out
  env ${kv//,/ } timeout 600 python scripts/kbench.py --cases $K >> $out 2>&1
done
