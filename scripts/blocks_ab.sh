# source blocking: parity + sweep of the block size on cfg5, regression check elsewhere
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/blocks_ab.log; rm -f $o
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_blocks.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_blocks.log
echo "== default" >> $o; timeout 600 python scripts/kbench.py --cases ${KC:-er128,rmat256,rmat100sym,rmat512h,cfg5mean} >> $o 2>&1
for mb in ${MBS:-24 32 64 96 160 100000}; do echo "== block_mb $mb" >> $o; GSPMM_SRC_BLOCK_MB=$mb timeout 600 python scripts/kbench.py --cases cfg5mean >> $o 2>&1; done
