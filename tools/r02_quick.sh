# quick GPU check of selected tests (PYTEST_K) + the cfg1 bench line
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -q -m gpu -x -k "${PYTEST_K:-step_host}" 2>&1 | tail -2
timeout 600 python bench.py --config cfg1 --steps 200 --warmup 10 > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/r02_bench_cfg1.err; echo cfg1 rc=$?
tail -2 gpurun_out/r02_bench_cfg1.err
