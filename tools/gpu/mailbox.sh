# analysis with mailbox read-backs vs B2L_NO_MAILBOX: parity subset, device-resident timing,
# interference with a concurrent upload, analyze_many e2e through bench.py
timeout 900 python -m pytest tests -m gpu -x -q -k "analysis or savings or standalone or reports or parity or sort" 2>&1 | tail -2
for mb in on off; do
  if [ $mb = off ]; then export B2L_NO_MAILBOX=1; fi
  echo "== mailbox $mb"
  for cfg in "c2 10000 30" "c2 1000000 30" "c2 10000000 8"; do
    set -- $cfg; timeout 300 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
  done
  timeout 300 python tools/pipe_exp3.py 2>&1 | head -2
  timeout 600 python bench.py --no-cpu --no-large --no-configs --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); a=d['analysis']; print('bench analysis', a['value'], 'e2e', a['e2e']['value'], a['e2e'].get('single_call'))"
done
