# r04d: split_edges parity test; cfg3 bench step default vs --split-edges 512 (with --verify)
O=gpurun_out/r04d
mkdir -p $O
timeout 900 python -m pytest -x -q tests/test_parity_gpu.py -k "split_by_edges or dependent_pair" > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -15 $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-e2e --verify --split-edges 512 > $O/bench_cfg3_split512.json 2> $O/bench_cfg3_split512.log
echo "bench split rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg3_split512.json')); print(d['ms_per_step'], d['passes_ms'], d.get('verify'))"
timeout 900 python bench.py --steps 10 --warmup 3 --skip-cpu --skip-e2e --verify > $O/bench_cfg3.json 2> $O/bench_cfg3.log
echo "bench rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg3.json')); print(d['ms_per_step'], d['passes_ms'], d.get('verify'))"
