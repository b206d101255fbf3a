# fused front variants (items per thread, rows per load batch, CTAs per SM), prebuilt in tools/_exp
cp paper_2601_12713_b200/libb2l.so /tmp/libb2l_keep.so
for v in fb f842 f823 f814 fb f842; do
  cp tools/_exp/libb2l_$v.so paper_2601_12713_b200/libb2l.so
  echo "== $v"
  timeout -k 5 300 python -m pytest tests/test_analysis_gpu.py -q -x 2>&1 | tail -1
  for cfg in "c2 1000000 24" "c2 10000000 8"; do
    set -- $cfg
    timeout -k 5 300 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
  done
  B2L_TRACE=ev timeout -k 5 300 python tools/evlog.py --n 10000000 --iters 4 2>&1 | grep "validate"
done
cp /tmp/libb2l_keep.so paper_2601_12713_b200/libb2l.so
