# ncu evidence for the bench's kernels (run alone: ncu replays each kernel).
# Launch order per step: fwd k_gather / k_long_ws, then bwd; 3 warm-up steps.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e"
$B > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
for k in gather long; do for pass in fwd:6 bwd:7; do
  ncu --set full --import-source on --clock-control none -k regex:k_$k -s ${pass#*:} -c 1 \
      -o gpurun_out/prof_${k}_${pass%:*} python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e \
      > gpurun_out/ncu_full_${k}_${pass%:*}.log 2>&1
done; done
echo "rc=$?" >> gpurun_out/ncu_full_long_bwd.log
