# Round-1 final pass: MX8 tests (diag pass templated), default bench (with variants), wall time
set -x
timeout 1200 python -m pytest tests/test_gpu_mx8.py -q -x > gpurun_out/pytest_mx8.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_mx8.log
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$? wall=$(( $(date +%s) - t0 ))
python bench.py --weights mx8 > gpurun_out/bench_cfg3_mx8.log 2>&1; echo mx8=$?
python bench.py --weights mx8 --storage dedup > gpurun_out/bench_cfg3_mx8_dedup.log 2>&1; echo mx8d=$?
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:superpose_mx8_mixed -s 2 -c 1 -f -o gpurun_out/superpose_mx8_dedup_cfg3 \
    python bench.py --weights mx8 --storage dedup --steps 3 --warmup 3 --no-cpu-baseline --no-variants --e2e-steps 2 --no-kgen-median > gpurun_out/ncu_mx8d.log 2>&1; echo ncu=$?
