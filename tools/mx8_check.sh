# MX8 weight format: GPU parity + bench line + ncu of the superposition kernel
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mx8.py -x -q > gpurun_out/pytest_mx8.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_mx8.log
timeout 600 python bench.py --weights mx8 --no-variants --no-cpu-baseline > gpurun_out/bench_mx8.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_mx8.log | cut -c1-1500
timeout 600 ncu --set full --clock-control none --import-source on -k regex:superpose_mx8 -c 1 -o gpurun_out/superpose_mx8_cfg3 -f \
  python bench.py --weights mx8 --no-variants --no-cpu-baseline --steps 2 --warmup 1 --e2e-steps 2 --no-kgen-median > gpurun_out/ncu_mx8.log 2>&1; echo ncu=$?
