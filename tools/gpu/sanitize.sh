# compute-sanitizer over small invocations of every kernel path (analysis, sorts, sharding, hash K1/K2)
CS="compute-sanitizer --print-limit 5"
for tool in memcheck racecheck synccheck; do
  echo "== ${tool}_analysis"; timeout 900 $CS --tool $tool python tools/sanitize_small.py 3000 2>&1 | grep -E "^ok|SUMMARY|Error|error" | head -8
done
echo "== memcheck_hash"; timeout 900 $CS --tool memcheck python -m pytest tests/test_hash_gpu.py -q -k "k2_small or golden or offsets" 2>&1 | grep -E "passed|failed|SUMMARY" | head -4
echo "== racecheck_hash"; timeout 900 $CS --tool racecheck python -m pytest tests/test_hash_gpu.py -q -k "k2_small" 2>&1 | grep -E "passed|failed|SUMMARY" | head -4
echo "== memcheck_hash_routes"; timeout 900 $CS --tool memcheck python -m pytest tests/test_hash_gpu.py tests/test_capture.py -q -k "single_buffer_routing or device_copy or every_length" 2>&1 | grep -E "passed|failed|SUMMARY" | head -4
