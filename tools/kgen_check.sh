python tools/kgen_timing.py cfg5 3 > gpurun_out/kgen_cfg5.txt 2>&1; cat gpurun_out/kgen_cfg5.txt
python tools/kgen_timing.py cfg3 3 > gpurun_out/kgen_cfg3.txt 2>&1; cat gpurun_out/kgen_cfg3.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
