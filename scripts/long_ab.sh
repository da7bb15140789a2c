cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/long_ab.log
for c in 0 24 40 64; do
  echo "== GSPMM_LONG_CTAS=$c" >> gpurun_out/long_ab.log
  GSPMM_LONG_CTAS=$c timeout 300 python scripts/kbench.py --cases rmat256,rmat512h,rmat100sym >> gpurun_out/long_ab.log 2>&1
done
timeout 300 python scripts/kbench.py --cases star256 >> gpurun_out/long_ab.log 2>&1
GSPMM_UNIT_TRACE=gpurun_out/trace6.bin timeout 300 python scripts/kbench.py --cases star256 > /dev/null 2>&1
GSPMM_UNIT_TRACE=gpurun_out/trace7.bin timeout 300 python scripts/kbench.py --cases rmat100sym > /dev/null 2>&1
