# ncu --set full of the edge-destined dot kernel on the cfg2 / cfg4 shapes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in ${DC:-cfg2dot}; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dot_edges -s 2 -c 1 \
   -o gpurun_out/prof_$c python scripts/kbench.py --cases $c > gpurun_out/ncu_$c.log 2>&1
done
