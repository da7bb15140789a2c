# ncu --set full of the row kernels on chosen kbench cases (one launch each)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in ${NC:-cfg5mean cfg3max}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather -s 2 -c 1 \
     -o gpurun_out/prof_${c}_g python scripts/kbench.py --cases $c > gpurun_out/ncu_${c}_g.log 2>&1
done
