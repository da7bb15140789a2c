# The parity case and the planned-kernel parity tests against a
# -DGSPMM_BOUNDS=1 build (device asserts on every gathered row id, output row,
# stage offset and id-ring slot; gather_impl.cuh): a failed assert traps the
# kernel and the run fails with a CUDA error.
#   make -C paper_2007_06354_b200 BUILD=_build_bc LIB=_ab/bounds.so EXTRA=-DGSPMM_BOUNDS=1
O=gpurun_out/bounds
mkdir -p $O
cp paper_2007_06354_b200/_lib/libgspmm_b200.so /tmp/intree.so
cp paper_2007_06354_b200/_ab/bounds.so paper_2007_06354_b200/_lib/libgspmm_b200.so
timeout 600 python scripts/sanitize_case.py > $O/sanitize_case.log 2>&1; echo "sanitize_case rc=$?"; tail -1 $O/sanitize_case.log
timeout 1500 python -m pytest -x -q tests/test_parity_gpu.py tests/test_concurrency_gpu.py > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 900 python scripts/kb_cfg3.py - > $O/kb_cfg3.jsonl 2> $O/kb_cfg3.err; echo "cfg3 passes rc=$?"; cat $O/kb_cfg3.jsonl
cp /tmp/intree.so paper_2007_06354_b200/_lib/libgspmm_b200.so
