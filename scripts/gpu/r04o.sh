# r04o: e2e of the default bench again, with the PCIe probe beside it
O=gpurun_out/r04o
mkdir -p $O
timeout 300 python scripts/pcie_bw.py > $O/pcie.txt 2>&1; tail -6 $O/pcie.txt
timeout 900 python bench.py --steps 10 --warmup 3 --skip-cpu > $O/bench_cfg3.json 2> $O/bench_cfg3.log
echo "bench rc=$?"; python -c "
import json; d=json.load(open('$O/bench_cfg3.json')); print(d['ms_per_step'], d['passes_ms'], d['e2e']['ms_per_step'])"
timeout 300 python scripts/pcie_bw.py > $O/pcie2.txt 2>&1; tail -6 $O/pcie2.txt
