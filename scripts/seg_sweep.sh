# sweep: segment unit cost (GSPMM_SEG_EDGES)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/seg_sweep.log; rm -f $o
for se in ${SES:-1024 256 512 2048}; do echo "== seg_edges $se" >> $o; GSPMM_SEG_EDGES=$se timeout 600 python scripts/kbench.py --cases ${KC:-er256,rmat256,cfg2bwd,rmat100sym,rmat512h} >> $o 2>&1; done
