timeout 900 python -m pytest tests/test_analysis_gpu.py -x -q 2>&1 | tail -40 > gpurun_out/ana_tests.log
cat gpurun_out/ana_tests.log
