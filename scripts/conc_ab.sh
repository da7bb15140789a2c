# kbench (ws vs g4 long rows) + concurrent traces after the dynamic first-unit change
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/conc_ab.log; rm -f $o
C=${KC:-er128,rmat256,rmat100sym,cfg3max,rmat512h,cfg5mean}
for k in ws g4; do echo "== kbench $k" >> $o; GSPMM_LONG_KERNEL=$k timeout 600 python scripts/kbench.py --cases $C >> $o 2>&1; done
for c in ${TC:-rmat256 rmat100sym}; do for k in ws g4; do echo "== trace $c $k" >> $o; GSPMM_LONG_KERNEL=$k timeout 200 python scripts/trace_conc.py $c 2>&1 | grep -v "^{" >> $o; done; done
