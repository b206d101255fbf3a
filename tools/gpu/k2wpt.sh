# K2 words per thread x CTAs per SM (prebuilt into tools/_exp with -DK2_WPT / -DK2_MIN_BLOCKS)
cp paper_2601_12713_b200/libb2l.so /tmp/libb2l_keep.so
for v in w24 w32 w36 w48; do
  cp tools/_exp/libb2l_$v.so paper_2601_12713_b200/libb2l.so
  echo "== $v"
  timeout -k 5 200 python -m pytest tests/test_hash_gpu.py -q -x -k "k2 or large or routing" 2>&1 | tail -1
  timeout -k 5 200 python tools/k2_time.py $((256<<20)) $((1<<20))
done
cp /tmp/libb2l_keep.so paper_2601_12713_b200/libb2l.so
