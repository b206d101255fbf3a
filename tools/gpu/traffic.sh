# analysis DRAM/L2 traffic per step at 1M and 10M events (every kernel of one analyze+savings step)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
for n in 1000000 10000000; do
  timeout -k 10 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/traffic_c2_$n.csv python tools/time_analysis.py --device --config c2 --n $n --iters 2 > /dev/null 2>&1
  python tools/analysis_traffic.py gpurun_out/traffic_c2_$n.csv 2 $n gpurun_out/analysis_traffic_c2_$n.json > /dev/null
done
for cfg in "c2 1000000 20" "c2 10000000 8" "c4 10000000 8"; do
  set -- $cfg
  timeout -k 10 600 python tools/time_analysis.py --device --config $1 --n $2 --iters $3 2>&1 | tail -1
done
