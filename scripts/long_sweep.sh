# sweep: forced long-row threshold (single plan level)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/long_sweep.log; rm -f $o
echo "== auto" >> $o; timeout 600 python scripts/kbench.py --cases ${KC:-rmat256,cfg2bwd,rmat100sym,rmat512h} >> $o 2>&1
for le in ${LES:-1024 2048 4096 8192}; do echo "== long_edges $le" >> $o; GSPMM_LONG_EDGES=$le timeout 600 python scripts/kbench.py --cases ${KC:-rmat256,cfg2bwd,rmat100sym,rmat512h} >> $o 2>&1; done
