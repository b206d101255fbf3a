# full GPU tests, smoke, bench, analysis traffic (1M, 10M), hash launch list
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
for n in 1000000 10000000; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/traffic_c2_$n.csv python tools/time_analysis.py --device --config c2 --n $n --iters 2 > /dev/null 2>&1
  python tools/analysis_traffic.py gpurun_out/traffic_c2_$n.csv 2 $n gpurun_out/analysis_traffic_c2_$n.json > /dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/hash_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-large > gpurun_out/bench_ncu.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 2500 gpurun_out/bench.log; tail -c 600 gpurun_out/bench_ref.log
