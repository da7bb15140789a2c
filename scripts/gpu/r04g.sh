# r04g: cfg3 step with the independent backward passes on two streams
O=gpurun_out/r04g
mkdir -p $O
timeout 900 python scripts/overlap_bwd.py > $O/overlap.jsonl 2> $O/overlap.err
echo rc=$?; cat $O/overlap.jsonl; tail -3 $O/overlap.err
