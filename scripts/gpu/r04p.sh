# r04p: e2e of the cfg3 bench, the previous hand-out order (_ab/old.so) against the new one, alternating
O=gpurun_out/r04p
mkdir -p $O
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/new.so
for i in 1 2; do
  for v in old new; do
    if [ $v = old ]; then cp paper_2007_06354_b200/_ab/old.so paper_2007_06354_b200/_lib/libgspmm_b200.so; else cp /tmp/new.so paper_2007_06354_b200/_lib/libgspmm_b200.so; fi
    timeout 900 python bench.py --steps 5 --warmup 3 --skip-cpu > $O/bench_${v}_$i.json 2> $O/bench_${v}_$i.log
    python -c "
import json; d=json.load(open('$O/bench_${v}_$i.json')); print('$v', $i, d['ms_per_step'], d['passes_ms'], d['e2e']['ms_per_step'])"
  done
done
cp /tmp/new.so paper_2007_06354_b200/_lib/libgspmm_b200.so
free -g | head -3; nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.width.current --format=csv
