# chains on three streams at large traces? (B2L_OVERLAP_MAX)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in "c2 10000000 8" "c4 10000000 8" "c2 30000000 5" "c2 100000000 5"; do
  set -- $cfg
  echo "== $cfg default";  timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
  echo "== $cfg overlap"; B2L_OVERLAP_MAX=1000000000 timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
