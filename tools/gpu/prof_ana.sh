# ncu --set full on the top analysis kernels (C2 10M), one instance each (after warm-up)
prof() {  # name regex skip
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$2" --launch-skip $3 -c 1 -o gpurun_out/prof_$1 -f python tools/time_analysis.py --device --config c2 --n 10000000 --iters 3 > /dev/null 2>&1
}
prof qop_scan "QOp" 1
prof onesweep1 "k_onesweep" 30

prof attr_pairs "ElemPairs" 1
ls gpurun_out/prof_*
