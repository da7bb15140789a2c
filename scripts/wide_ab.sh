# wide (VPL 5) segment units: parity + cfg5 kbench (wide on / off) + the cfg5 bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/wide_ab.log; rm -f $o
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_wide.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wide.log
echo "== wide" >> $o; timeout 600 python scripts/kbench.py --cases cfg5mean,rmat256 >> $o 2>&1
echo "== nowide" >> $o; GSPMM_WIDE_UNITS=0 timeout 600 python scripts/kbench.py --cases cfg5mean >> $o 2>&1
for mb in 32 64; do echo "== wide block_mb $mb" >> $o; GSPMM_SRC_BLOCK_MB=$mb timeout 600 python scripts/kbench.py --cases cfg5mean >> $o 2>&1; done
timeout 900 python bench.py --workload cfg5 --steps 5 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
