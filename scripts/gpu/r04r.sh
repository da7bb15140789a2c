# r04r: edge softmax with rows handed out from a counter: tests and timings
O=gpurun_out/r04r
mkdir -p $O
timeout 900 python -m pytest -x -q tests/test_softmax_gpu.py tests/test_concurrency_gpu.py tests/test_autograd_gpu.py > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 900 python scripts/kbench.py --cases cfg4softmax,cfg4softmaxbwd > $O/kbench.jsonl 2> $O/kbench.err
cut -c1-200 $O/kbench.jsonl
