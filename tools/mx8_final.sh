# MX8 final pass: GPU parity, bench lines (cfg3 / cfg5), compute-sanitizer memcheck + synccheck
set -x
timeout 900 python -m pytest tests/test_gpu_mx8.py -x -q > gpurun_out/pytest_mx8.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_mx8.log
python bench.py --weights mx8 > gpurun_out/bench_cfg3_mx8.log 2>&1; tail -1 gpurun_out/bench_cfg3_mx8.log | cut -c1-300
python bench.py --config cfg5 --weights mx8 --steps 100 --no-variants > gpurun_out/bench_cfg5_mx8.log 2>&1; tail -1 gpurun_out/bench_cfg5_mx8.log | cut -c1-300
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(tail -2 gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
