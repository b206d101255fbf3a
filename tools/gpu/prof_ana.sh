# ncu --set full on the top analysis kernels (C2 10M), one instance each (after warm-up)
prof() {  # name regex skip
  timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$2" --launch-skip $3 -c 1 -o gpurun_out/prof_$1 -f python tools/time_analysis.py --device --config c2 --n 10000000 --iters 3 > /dev/null 2>&1
}
prof qop_scan "k_scan_1p<ana::QOp" 1
prof onesweep1 "k_onesweep<1>" 30
prof front_reduce "k_front_reduce" 1
prof attr_pairs "k_attr<ana::ElemPairs>" 1
ls gpurun_out/prof_*
timeout 900 python -m pytest tests/test_hash_gpu.py -q -x 2>&1 | grep -E "^E  |passed|failed" | head -20
timeout 300 python tools/bench_configs.py --configs c3 2>&1 | head -1
