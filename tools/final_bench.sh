# final bench refresh: default cfg3 (with variants), cfg5 bf16, cfg5 mx8, reference arm
python bench.py > gpurun_out/bench_cfg3.log 2>&1; echo cfg3=$?
python bench.py --config cfg5 --steps 100 > gpurun_out/bench_cfg5.log 2>&1; echo cfg5=$?
python bench.py --config cfg5 --weights mx8 --steps 100 --no-variants > gpurun_out/bench_cfg5_mx8.log 2>&1; echo cfg5mx8=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
