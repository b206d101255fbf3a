# fused single-pass front vs the two-pass reduce/apply: GPU tests, then timings
timeout -k 10 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for mode in fused two; do
  if [ $mode = two ]; then export B2L_FRONT_TWO_PASS=1; fi
  echo "== $mode"
  for cfg in "c2 1000000 24" "c2 10000000 8" "c4 10000000 8"; do
    set -- $cfg
    timeout -k 5 300 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
  done
done
unset B2L_FRONT_TWO_PASS
B2L_TRACE=ev timeout -k 5 300 python tools/evlog.py --n 10000000 --iters 4 2>&1 | sed -n '/=== last call/,$p' | head -6
