# host-vs-GPU phase timeline of one warm analyze call at 10M and 1M events (C2)
B2L_TRACE=ev timeout -k 5 300 python tools/evlog.py --n 10000000 --iters 4 2>&1 | sed -n '/=== last call/,$p' > gpurun_out/evlog_10m.txt
B2L_SYNC_STATS=2 B2L_TRACE=ev timeout -k 5 300 python tools/evlog.py --n 1000000 2>&1 | sed -n '/=== last call/,$p' > gpurun_out/evlog_1m.txt
cat gpurun_out/evlog_10m.txt
