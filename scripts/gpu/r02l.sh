# r02l: the container loaders on the GPU, the C++ shim harness with the io
# checks, then compute-sanitizer over every kernel family.
mkdir -p gpurun_out/r02l
timeout 900 python -m pytest -x -q tests/test_io_gpu.py tests/test_shim_cpp.py > gpurun_out/r02l/pytest.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/r02l/pytest.log
bash scripts/gpu/sanitize.sh
