# Round-1 profiling pass (one GPU): launch list of the bench command, ncu --set full of the
# dominant step kernel (superpose_bulk_kernel, cfg3) and of kgen (Chebyshev, cfg3).  Outputs in gpurun_out/.
set -x
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:kgen_kernel -s 1 -c 1 -f -o gpurun_out/kgen_cfg3 \
    python tools/kgen_timing.py cfg3 2 0 > gpurun_out/ncu_kgen.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:superpose_bulk_kernel -s 2 -c 1 -f -o gpurun_out/superpose_cfg3 \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/ncu_sup.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:superpose_mixed_bulk_kernel -s 2 -c 1 -f -o gpurun_out/superpose_n4_cfg3 \
    python bench.py --storage dedup --steps 3 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/ncu_sup_n4.log 2>&1
python bench.py > gpurun_out/bench_cfg3.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
python bench.py --config cfg5 --steps 100 > gpurun_out/bench_cfg5.log 2>&1
python bench.py --config cfg2 --steps 500 > gpurun_out/bench_cfg2.log 2>&1
ls -la gpurun_out
