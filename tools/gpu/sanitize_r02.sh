# compute-sanitizer over the round-2 kernel paths: split pairs + dynamic claims (ragged batches),
# merged host copy runs, mailbox read-backs + zeroed scratch pool (analysis), sharded routing
CS="compute-sanitizer --print-limit 5"
for tool in memcheck racecheck synccheck; do
  echo "== ${tool}_split_pairs"; timeout 900 $CS --tool $tool python -m pytest tests/test_hash_gpu.py -q -k "split_pairs or ragged_longest" 2>&1 | grep -E "passed|failed|SUMMARY" | head -4
done
echo "== memcheck_host_runs"; timeout 900 $CS --tool memcheck python -m pytest tests/test_hash_gpu.py -q -k "merged_copy_runs" 2>&1 | grep -E "passed|failed|SUMMARY" | head -4
for tool in memcheck racecheck synccheck; do
  echo "== ${tool}_analysis"; timeout 900 $CS --tool $tool python tools/sanitize_small.py 3000 --no-sharded 2>&1 | grep -E "^ok|SUMMARY|Error|error" | head -8
done
echo "== memcheck_sharded"; timeout 900 $CS --tool memcheck python tools/sanitize_small.py 3000 2>&1 | grep -E "^ok|SUMMARY|Error|error" | head -8
