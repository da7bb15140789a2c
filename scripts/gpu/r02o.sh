# r02o: ncu --set full of the long-row kernel (sum variant, then the DUAL variant) on cfg3
mkdir -p gpurun_out/r02o
O=gpurun_out/r02o
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_long_rg --launch-skip 14 -c 1 -o $O/long_sum python scripts/kb_cfg3.py - > $O/ncu1.log 2>&1
echo ncu1 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_long_rg --launch-skip 27 -c 1 -o $O/long_dual python scripts/kb_cfg3.py - > $O/ncu2.log 2>&1
echo ncu2 rc=$?
ls -la $O
