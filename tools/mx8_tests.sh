timeout 1200 python -m pytest tests/test_gpu_mx8.py -q > gpurun_out/pytest_mx8.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_mx8.log | grep -v "^$" | tail -20
for v in "FDIRW_MX8_NSUB=1" ""; do echo "== $v"; env $v python bench.py --config cfg2 --weights mx8 --steps 500 --no-variants --no-cpu-baseline --e2e-steps 5 --no-kgen-median 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"; done
python bench.py --config cfg2 --weights mx8 --steps 500 --no-variants > gpurun_out/bench_cfg2_mx8.log 2>&1
