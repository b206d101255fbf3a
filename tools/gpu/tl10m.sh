# warm timelines of the 1M and 10M steps, per stream (where the critical chain waits)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out
timeout 600 python tools/timeline.py --config c2 --n 10000000 --streams > gpurun_out/tl10m.txt 2>&1
timeout 600 python tools/timeline.py --config c2 --n 1000000 --streams > gpurun_out/tl1m.txt 2>&1
timeout 600 python tools/timeline.py --config c4 --n 10000000 > gpurun_out/tl_c4_10m.txt 2>&1
tail -3 gpurun_out/tl10m.txt
