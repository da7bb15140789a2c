# r02w: cfg4 / cfg2 passes under plan variants (did the column-unit long-row kernel cost cfg4?),
# the new long-row tie / zero / NaN test, zero-width operands, e2e with per-call streams
O=gpurun_out/r02w
mkdir -p $O
timeout 600 python -m pytest -x -q tests/test_parity_gpu.py -k "ties_zeros or validation or empty" > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 900 python scripts/kbench.py --cases rmat512h,cfg4bwdx,rmat256 --plans "/ long_ctas=74 / long_ctas=32 / unit_cols=128 / unit_cols=512 / long_threshold=16384 / long_threshold=65536" > $O/kb.jsonl 2> $O/kb.err
cat $O/kb.jsonl
timeout 900 python bench.py --steps 5 --warmup 3 --skip-cpu > $O/bench_cfg3.json 2> $O/bench_cfg3.log
echo "bench rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg3.json')); print(d['ms_per_step'], d['e2e'])"
