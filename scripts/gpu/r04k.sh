# r04k: last check of the final HEAD's library: smoke, the parity and concurrency suites, the
# driver's bench command with default flags
O=gpurun_out/r04k
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_concurrency_gpu.py tests/test_softmax_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest.log
SECONDS=0
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.log
echo "bench rc=$? wall ${SECONDS}s"; python -c "
import json; d=json.load(open('$O/bench_default.json')); print(d['ms_per_step'], d['value']/1e9, d['e2e']['ms_per_step'], d['roofline']['frac'], d['roofline']['dram_frac'], d['clocks'], d['gpu_launches'], d['steps'])"
