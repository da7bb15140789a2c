# ncu evidence for the bench's kernels (run alone: ncu replays each kernel)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e \
    > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_gather -s 6 -c 1 \
    -o gpurun_out/prof_gather python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e \
    > gpurun_out/ncu_full.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k_long -s 6 -c 1 \
    -o gpurun_out/prof_long python bench.py --steps 1 --warmup 3 --skip-cpu --skip-e2e \
    > gpurun_out/ncu_full2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full2.log
