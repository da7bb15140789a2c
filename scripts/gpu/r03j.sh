# r03j: final check of HEAD: GPU suite, smoke, default bench line (csv rows included)
O=gpurun_out/r03j
mkdir -p $O
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.log
echo "bench rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg3.json')); print(d['ms_per_step'], d['e2e']['ms_per_step']); print('\n'.join(d['csv']))"
