# ncu --set full of the heaviest analysis kernels on the 10M-event C2 trace (one launch each)
set -x
for k in "ElemPairs" "RtMaxLoad" "QOp" "k_onesweep<1, 16>" "k_front_reduce" "DepthLoad"; do
  tag=$(echo "$k" | tr -dc 'A-Za-z0-9')
  timeout 600 ncu --set full --clock-control none --kernel-name-base demangled \
    -k "regex:.*${k}.*" -c 1 -o gpurun_out/p10m_$tag -f \
    python tools/time_analysis.py --device --config c2 --n 10000000 --iters 2 > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep
