# one ncu --set full capture of the long-row kernel for a kbench case
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
C=${C:-rmat256}
GSPMM_LONG_ASYNC=1 timeout 300 python scripts/kbench.py --cases $C > gpurun_out/nl_plain.log 2>&1 && \
GSPMM_LONG_ASYNC=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_long -s 3 -c 1 \
  -o gpurun_out/nl_${C} python scripts/kbench.py --cases $C > gpurun_out/nl_full.log 2>&1
echo "rc=$?" >> gpurun_out/nl_full.log
