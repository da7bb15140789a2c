# sweep: long-row CTA count factor and XL slice width for the gather4 kernel
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/g4_sweep.log; rm -f $o
C=${KC:-rmat256,rmat512h}
for f in 30 45 60 90; do for x in 64 128; do
  echo "== g4 factor $f xl $x" >> $o
  GSPMM_LONG_FACTOR10=$f GSPMM_XL_SW=$x timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1
done; done
for f in 30 45; do echo "== ws factor $f" >> $o; GSPMM_LONG_KERNEL=ws GSPMM_LONG_FACTOR10=$f timeout 300 python scripts/kbench.py --cases $C >> $o 2>&1; done
