# MX8 profiling pass (one GPU): ncu --set full of superpose_mx8_kernel at cfg3, bench lines
# (default cfg3 with the mx8 variant; --weights mx8 at cfg3 / cfg2 / cfg5 / cfg4).  Outputs in gpurun_out/.
set -x
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:superpose_mx8 -s 2 -c 1 -f -o gpurun_out/superpose_mx8_cfg3 \
    python bench.py --weights mx8 --steps 3 --warmup 3 --no-cpu-baseline --no-variants --e2e-steps 2 --no-kgen-median > gpurun_out/ncu_mx8.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_mx8.csv \
    python bench.py --weights mx8 --steps 20 --warmup 3 --no-cpu-baseline --no-variants --no-kgen-median > gpurun_out/launches_mx8.log 2>&1
python bench.py --weights mx8 > gpurun_out/bench_cfg3_mx8.log 2>&1
python bench.py > gpurun_out/bench_cfg3.log 2>&1
python bench.py --config cfg2 --weights mx8 --steps 500 --no-variants > gpurun_out/bench_cfg2_mx8.log 2>&1
python bench.py --config cfg5 --weights mx8 --steps 100 --no-variants > gpurun_out/bench_cfg5_mx8.log 2>&1
timeout 900 python bench.py --config cfg4 --weights mx8 --steps 50 --no-variants --no-cpu-baseline > gpurun_out/bench_cfg4_mx8.log 2>&1
for f in gpurun_out/bench_*mx8*.log gpurun_out/bench_cfg3.log; do echo $f; tail -1 $f | cut -c1-300; done
