python bench.py --config cfg3o --weights mx8 --no-variants > gpurun_out/bench_cfg3o_mx8.log 2>&1; echo cfg3o=$?; tail -1 gpurun_out/bench_cfg3o_mx8.log | cut -c1-200
python bench.py --mode absorb --weights mx8 > gpurun_out/bench_absorb_mx8.log 2>&1; echo absorb=$?; tail -1 gpurun_out/bench_absorb_mx8.log | cut -c1-200
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
