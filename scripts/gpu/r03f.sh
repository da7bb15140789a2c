# r03f: bounds-checking build over the parity case, the planned-kernel tests and the cfg3 passes;
# cfg1 bench line with the in-process clock sample
bash scripts/gpu/bounds.sh
timeout 600 python bench.py --workload cfg1 --steps 20 --warmup 3 --skip-cpu > gpurun_out/bounds/bench_cfg1.json 2> gpurun_out/bounds/bench_cfg1.log
echo "bench cfg1 rc=$?"; cut -c1-900 gpurun_out/bounds/bench_cfg1.json
