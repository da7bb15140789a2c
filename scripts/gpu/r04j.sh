# r04j: --set full of the edge-softmax kernels on the cfg4 shape
O=gpurun_out/r04j
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_softmax --launch-skip 8 -c 4 -o $O/softmax python scripts/kbench.py --cases cfg4softmax,cfg4softmaxbwd > $O/ncu.log 2>&1
echo rc=$?; tail -3 $O/ncu.log
