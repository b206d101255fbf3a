cp paper_2601_12713_b200/libb2l.so /tmp/keep.so
for v in cur t192w48 t288w32; do
  cp tools/_exp/libb2l_$v.so paper_2601_12713_b200/libb2l.so
  echo "== $v"
  timeout -k 5 200 python -m pytest tests/test_hash_gpu.py -q -x -k "k2 or large or routing" 2>&1 | tail -1
  timeout -k 5 200 python tools/k2_time.py $((256<<20)) 2>&1 | grep -E "K2"
done
cp /tmp/keep.so paper_2601_12713_b200/libb2l.so
