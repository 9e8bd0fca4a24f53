timeout 1200 python -m pytest tests/test_gpu_mx8.py -q -x > gpurun_out/pytest_mx8.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_mx8.log
