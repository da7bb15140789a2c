# r04n: parity after the hand-out order change; the default bench line
O=gpurun_out/r04n
mkdir -p $O
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py tests/test_concurrency_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --skip-cpu > $O/bench_cfg3.json 2> $O/bench_cfg3.log
echo "bench rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg3.json')); print(d['ms_per_step'], d['passes_ms'], d['e2e']['ms_per_step'])"
