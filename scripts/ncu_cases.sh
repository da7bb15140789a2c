# ncu evidence for kbench cases: launch list + one full capture of the
# segment kernel and the long-row kernel per case (run alone on one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CASES=${CASES:-cfg3max,cfg5mean,rmat512h}
for k in ${CASES//,/ }; do
  timeout 300 python scripts/kbench.py --cases $k > gpurun_out/nc_$k.plain.log 2>&1 || { echo "plain $k failed" >> gpurun_out/nc_$k.plain.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/nc_$k.launches.csv python scripts/kbench.py --cases $k > /dev/null 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather -s 3 -c 1 \
    -o gpurun_out/nc_${k}_gather python scripts/kbench.py --cases $k > gpurun_out/nc_$k.full.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_long -s 3 -c 1 \
    -o gpurun_out/nc_${k}_long python scripts/kbench.py --cases $k >> gpurun_out/nc_$k.full.log 2>&1
done
echo done > gpurun_out/nc_done
