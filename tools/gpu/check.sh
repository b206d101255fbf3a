# GPU tests + smoke + bench (N=1) + reference arm
set -x
timeout -k 10 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout -k 10 900 python bench.py > gpurun_out/bench.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 3000 gpurun_out/bench.log
