# K2 spin back-off sweep (variants prebuilt into tools/_exp with -DK2_SPIN_NS=...)
cp paper_2601_12713_b200/libb2l.so /tmp/libb2l_keep.so
for ns in 0 64 400; do
  cp tools/_exp/libb2l_s$ns.so paper_2601_12713_b200/libb2l.so
  timeout -k 5 200 python -m pytest tests/test_hash_gpu.py -q -x -k "k2 or large or routing" 2>&1 | tail -1
  cp tools/_exp/libb2l_s$ns.so paper_2601_12713_b200/libb2l.so
  echo "== spin $ns ns"
  K2_MANY=0 timeout -k 5 120 python tools/k2_time.py $((256<<20)) $((16<<20)) $((1<<20))
  B2L_K2_JOBS=16 timeout -k 5 120 python tools/k2_time.py 0 2>&1 | grep many
  B2L_K2_JOBS=8 B2L_K2_TEAMS=2 timeout -k 5 120 python tools/k2_time.py 0 2>&1 | grep "many"
done
cp /tmp/libb2l_keep.so paper_2601_12713_b200/libb2l.so
