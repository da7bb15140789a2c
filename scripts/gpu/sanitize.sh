# compute-sanitizer over every kernel family on small graphs.
O=gpurun_out/sanitize
mkdir -p $O
timeout 300 python scripts/sanitize_case.py > $O/plain.log 2>&1; echo "plain rc=$?"; tail -1 $O/plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 66 --log-file $O/$tool.log python scripts/sanitize_case.py > $O/$tool.out 2>&1
  echo "$tool rc=$?"; tail -1 $O/$tool.out; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $O/$tool.log | tail -2
done
