# A/B of the streaming kernel's staging modes (development)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/stage_ab.log
for m in 0 512 100000; do
  echo "== GSPMM_TMA_MIN_BYTES=$m" >> gpurun_out/stage_ab.log
  GSPMM_TMA_MIN_BYTES=$m timeout 300 python scripts/kbench.py --cases ${KCASES:-star256,er256,rmat256,er128} >> gpurun_out/stage_ab.log 2>&1
done
