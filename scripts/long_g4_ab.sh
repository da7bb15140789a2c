# A/B of the long-row kernels (gather4 TMA default vs LDGSTS ws) + parity
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/g4_ab.log; rm -f $o
C=${KC:-rmat256,rmat100sym,cfg3max,rmat512h}
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_g4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g4.log
echo "== g4" >> $o; timeout 600 python scripts/kbench.py --cases $C >> $o 2>&1
echo "== ws" >> $o; GSPMM_LONG_KERNEL=ws timeout 600 python scripts/kbench.py --cases $C >> $o 2>&1
for c in rmat256 rmat100sym; do echo "== trace g4 $c" >> $o; timeout 200 python scripts/trace_case.py $c 2>&1 | tail -8 >> $o; done
