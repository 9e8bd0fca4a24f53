timeout 1200 python -m pytest tests/test_gpu_mx8.py -q -x > gpurun_out/pytest_mx8.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_mx8.log
python tools/slab_timing.py mx8 > gpurun_out/slab_mx8.txt 2>&1; cat gpurun_out/slab_mx8.txt
