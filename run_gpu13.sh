B2L_TRACE=1 timeout 300 python tools/time_analysis.py --device --iters 6 2>&1 | tail -30 | grep -E "detectors|partition|d2h|validate|upload|analyze|pairs|ra |ua_ut"
