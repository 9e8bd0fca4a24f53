timeout 1200 python -m pytest tests/test_gpu_mx8.py -q > gpurun_out/pytest_mx8.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_mx8.log | grep -v "^$" | tail -25
timeout 600 python -m pytest tests/test_gpu_far.py tests/test_gpu_absorb.py -q -x 2>&1 | tail -2
