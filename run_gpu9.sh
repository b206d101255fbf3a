CUDA_LAUNCH_BLOCKING=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/sanitize_small.py 5000 2>&1 | head -40
