# the remaining bench configs (one GPU): cfg3o (N2 far field), cfg4 on one GPU, cfg2 fp32, N1 coarse
python bench.py --config cfg3o --steps 300 --no-variants > gpurun_out/bench_cfg3o.log 2>&1
python bench.py --config cfg4 --steps 20 --warmup 3 --no-variants --no-cpu-baseline --e2e-steps 5 > gpurun_out/bench_cfg4.log 2>&1
python bench.py --config cfg2 --weights fp32 --steps 500 --no-variants --no-cpu-baseline > gpurun_out/bench_cfg2_fp32.log 2>&1
python bench.py --mode coarse --steps 300 --no-cpu-baseline > gpurun_out/bench_coarse.log 2>&1
python bench.py --mode coarse --config cfg3o --steps 300 --no-cpu-baseline > gpurun_out/bench_coarse_cfg3o.log 2>&1
for f in cfg3o cfg4 cfg2_fp32 coarse coarse_cfg3o; do echo $f; tail -1 gpurun_out/bench_$f.log | cut -c1-400; done
