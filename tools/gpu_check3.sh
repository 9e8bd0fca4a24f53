timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -8 gpurun_out/pytest_gpu.log
python tools/kgen_timing.py cfg3 2 0; python tools/kgen_timing.py cfg5 1 0
