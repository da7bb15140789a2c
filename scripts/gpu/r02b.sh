# r02b: first run of the column-unit long-row kernel, chunked argmax backward,
# per-stream call contexts; parity tests, then the cfg3 / cfg2 benches.
mkdir -p gpurun_out/r02b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu --deselect tests/test_scale_gpu.py > gpurun_out/r02b/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/r02b/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/r02b/bench_cfg3.json 2> gpurun_out/r02b/bench_cfg3.log
echo "bench cfg3 rc=$?"
timeout 600 python bench.py --workload cfg2 --steps 10 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/r02b/bench_cfg2.json 2> gpurun_out/r02b/bench_cfg2.log
echo "bench cfg2 rc=$?"
timeout 900 python -m pytest tests/test_scale_gpu.py -x -q > gpurun_out/r02b/pytest_scale.log 2>&1
echo "scale rc=$?"
tail -5 gpurun_out/r02b/pytest_scale.log
