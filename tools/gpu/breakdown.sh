# per-phase breakdown of the analysis pipeline at 10M / 100M events, plus a kernel launch list at 10M
for cfg in "c2 10000000" "c4 10000000" "c2 100000000"; do
  set -- $cfg
  B2L_TRACE=1 timeout 600 python tools/time_analysis.py --device --config $1 --n $2 --iters 3 2>&1 | tail -40 > gpurun_out/bd_$1_$2.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c2_10M.csv python tools/time_analysis.py --device --config c2 --n 10000000 --iters 1 > /dev/null 2>&1
timeout 300 python tools/time_analysis.py --device --config c2 --n 10000000 --iters 4 > gpurun_out/plain_c2_10M.log 2>&1
timeout 300 python tools/time_analysis.py --device --config c4 --n 10000000 --iters 4 > gpurun_out/plain_c4_10M.log 2>&1
ls -la gpurun_out
