# ncu --set full of the single-pass front at 10M events (C2)
timeout -k 10 900 ncu --set full --import-source on --clock-control none -k regex:k_front_fused -s 1 -c 1 -o gpurun_out/front_fused_10m -f python tools/time_analysis.py --device --config c2 --n 10000000 --iters 2 > gpurun_out/frontncu.log 2>&1
python tools/ncu_summary.py gpurun_out/front_fused_10m.ncu-rep gpurun_out/front_fused_10m_ncu_summary.json > /dev/null 2>&1
tail -3 gpurun_out/frontncu.log
