python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
B2L_SYNC_STATS=2 B2L_TRACE=ev timeout 300 python tools/evlog.py --n 1000000 2>&1 | sed -n '/=== last call/,$p' > gpurun_out/evlog_1m.txt
B2L_TRACE=ev timeout 300 python tools/evlog.py --n 10000 2>&1 | sed -n '/=== last call/,$p' > gpurun_out/evlog_10k.txt
cat gpurun_out/evlog_1m.txt
