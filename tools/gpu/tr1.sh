timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
B2L_TRACE=1 timeout 600 python tools/time_analysis.py --device --config c2 --n 1000000 --iters 6 2>&1 | tail -26
