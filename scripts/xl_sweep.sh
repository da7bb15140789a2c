# sweep: XL row threshold and forced long-row threshold
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/xl_sweep.log; rm -f $o
C=${KC:-rmat256,cfg2bwd}
for xe in 4096 8192 16384 32768; do echo "== xl_edges $xe" >> $o; GSPMM_XL_EDGES=$xe timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1; done
for le in 2048 4096 8192; do echo "== long_edges $le" >> $o; GSPMM_LONG_EDGES=$le timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1; done
