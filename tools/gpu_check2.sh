set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
python tools/kgen_timing.py cfg3 2 0; python tools/kgen_timing.py cfg3 1 32
python tools/kgen_timing.py cfg5 1 0; python tools/kgen_timing.py cfg5 1 32
python tools/kgen_timing.py cfg2 2 0
timeout 600 python bench.py --steps 100 --no-variants > gpurun_out/bench_cfg3.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_cfg3.log
