# round-end evidence: smoke, GPU tests, every kbench case, all bench workloads,
# ncu of the bench passes, the reference CPU path beside each configuration
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KCASES=er128,er256,rmat256,rmatcap256,rmat100sym,cfg3max,rmat512h,cfg5mean,cfg2dot,cfg4dot,cfg2bwd,cfg3meanbwd,cfg3maxbwd,cfg4bwdx,cfg5meanbwd,cfg4softmax,cfg4softmaxbwd bash scripts/gpu_check.sh
for w in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
bash scripts/ncu_bench.sh
timeout 2400 python scripts/cpu_ref.py --cases er128,rmat256,cfg2bwd,cfg2dot,rmat100sym,cfg3max,cfg3meanbwd,rmat512h,cfg4bwdx,cfg4dot,cfg5mean,cfg5meanbwd > gpurun_out/cpu_ref.jsonl 2> gpurun_out/cpu_ref.err
