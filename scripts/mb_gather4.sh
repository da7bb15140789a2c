# sweep of scripts/mb_gather4.cu (TMA gather4 long-row streaming rate per SM)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; o=gpurun_out/mb_gather4.log; rm -f $o
B=scripts/bin/mb_gather4
for cfg in "256 256 148 16384 32 4 4" "256 256 148 16384 48 4 4" "256 256 148 16384 48 4 0" "256 256 74 16384 48 4 4" \
           "256 64 148 32768 128 4 1" "256 64 148 32768 192 4 1" "256 64 148 32768 192 4 0" "256 64 148 32768 64 4 1" \
           "100 100 148 32768 96 4 4" "100 100 148 32768 128 4 4" "512 256 148 16384 48 4 4" "512 512 148 8192 24 4 4" \
           "256 128 148 32768 96 4 1" "256 256 8 16384 48 4 4" "256 64 8 32768 192 4 1"; do
  timeout 60 $B $cfg >> $o 2>&1 || echo "fail $cfg" >> $o
done
