CS="compute-sanitizer --print-limit 5"
echo "== racecheck_analysis (no sharded)"; timeout 1500 $CS --tool racecheck python tools/sanitize_small.py 3000 --no-sharded 2>&1 | grep -E "^ok|SUMMARY|Error|error" | head -8
