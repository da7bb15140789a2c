# sweep: forced long-row CTA count
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/ctas_sweep.log; rm -f $o
for c in ${CS:-24 37 50 74 100}; do echo "== long_ctas $c" >> $o; GSPMM_LONG_CTAS=$c timeout 600 python scripts/kbench.py --cases ${KC:-rmat256,cfg2bwd,rmat100sym,rmat512h} >> $o 2>&1; done
