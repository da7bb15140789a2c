# sweep: long-row CTA factor and XL slice width (ws long rows)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/ws_sweep.log; rm -f $o
C=${KC:-rmat256,cfg2bwd}
for f in ${FS:-20 30 45 60}; do for x in ${XS:-32 64 128}; do
  echo "== ws factor $f xl $x" >> $o
  GSPMM_LONG_FACTOR10=$f GSPMM_XL_SW=$x timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1
done; done
