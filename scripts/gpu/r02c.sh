mkdir -p gpurun_out/r02c
timeout 300 python scripts/mb_argmax_bwd.py > gpurun_out/r02c/mb.log 2>&1
cat gpurun_out/r02c/mb.log
timeout 600 ncu --set full -k regex:argmax -c 4 --import-source on -o gpurun_out/r02c/argmax python scripts/mb_argmax_bwd.py > gpurun_out/r02c/ncu.log 2>&1
echo ncu rc=$?
