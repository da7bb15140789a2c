cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/long_ab.log
for t in 0 4096 16384; do
  echo "== LONG_EDGES=$t" >> gpurun_out/long_ab.log
  GSPMM_LONG_EDGES=$t timeout 300 python scripts/kbench.py --cases rmat256,star256,rmat100sym,rmat512h,er256 >> gpurun_out/long_ab.log 2>&1
done
