# r04s: edge softmax, hub-row threshold sweep with the dynamic row hand-out
O=gpurun_out/r04s
mkdir -p $O
timeout 900 python scripts/kbench.py --cases cfg4softmax,cfg4softmaxbwd --plans " / long_threshold=2048 / long_threshold=4096 / long_threshold=8192 / long_threshold=16384" > $O/kbench.jsonl 2> $O/kbench.err
cut -c1-220 $O/kbench.jsonl
