mkdir -p gpurun_out/sanitizer
export PYTHONUNBUFFERED=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_hash_gpu.py -q -x -k "ts_vectors or misaligned_starts or ragged or zero_length or k2_small or audit" > gpurun_out/sanitizer/memcheck_hash.log 2>&1; tail -3 gpurun_out/sanitizer/memcheck_hash.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py 200000 > gpurun_out/sanitizer/memcheck_analysis.log 2>&1; tail -3 gpurun_out/sanitizer/memcheck_analysis.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py 20000 > gpurun_out/sanitizer/racecheck_analysis.log 2>&1; tail -3 gpurun_out/sanitizer/racecheck_analysis.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_small.py 20000 > gpurun_out/sanitizer/synccheck_analysis.log 2>&1; tail -3 gpurun_out/sanitizer/synccheck_analysis.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_hash_gpu.py -q -x -k "misaligned_starts_0_to_15 or k2_small" > gpurun_out/sanitizer/racecheck_hash.log 2>&1; tail -3 gpurun_out/sanitizer/racecheck_hash.log
