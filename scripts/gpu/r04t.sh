# r04t: final HEAD: whole GPU suite, smoke, the driver's two bench commands with default flags
O=gpurun_out/r04t
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?"; tail -1 $O/smoke.log
SECONDS=0
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.log
echo "bench rc=$? wall ${SECONDS}s"; python -c "
import json; d=json.load(open('$O/bench_default.json')); print(d['ms_per_step'], d['value']/1e9, d['passes_ms'], d['e2e']['ms_per_step'], d['e2e']['blocks_ms_per_step'], d['roofline']['frac'], d['roofline']['dram_frac'], d['clocks'], d['gpu_launches'], d['steps'])"
SECONDS=0
timeout 1200 python bench.py --impl reference > $O/bench_reference_default.json 2> $O/bench_reference_default.log
echo "ref rc=$? wall ${SECONDS}s"; cut -c1-300 $O/bench_reference_default.json
