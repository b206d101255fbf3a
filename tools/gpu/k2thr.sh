# K2 CTA-size variants (prebuilt into tools/_exp with -DK2_THREADS=...)
cp paper_2601_12713_b200/libb2l.so /tmp/libb2l_keep.so
for th in 128 512; do
  cp tools/_exp/libb2l_t$th.so paper_2601_12713_b200/libb2l.so
  echo "== threads $th"
  timeout -k 5 200 python -m pytest tests/test_hash_gpu.py -q -x -k "k2 or large or routing" 2>&1 | tail -1
  timeout -k 5 200 python tools/k2_time.py $((256<<20)) $((16<<20)) $((1<<20))
done
cp /tmp/libb2l_keep.so paper_2601_12713_b200/libb2l.so
