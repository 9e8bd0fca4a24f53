# every bench line committed under profiles/ (one GPU), written to gpurun_out/bench_<name>.log
python bench.py > gpurun_out/bench_cfg3.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
python bench.py --config cfg5 --steps 100 > gpurun_out/bench_cfg5.log 2>&1
python bench.py --config cfg2 --steps 500 > gpurun_out/bench_cfg2.log 2>&1
python bench.py --config cfg2 --weights fp32 --steps 500 --no-variants --no-cpu-baseline > gpurun_out/bench_cfg2_fp32.log 2>&1
python bench.py --config cfg1 --steps 100 > gpurun_out/bench_cfg1.log 2>&1
python bench.py --config cfg3o --steps 300 --no-variants > gpurun_out/bench_cfg3o.log 2>&1
python bench.py --config cfg4 --steps 20 --warmup 3 --no-variants --no-cpu-baseline --e2e-steps 5 --no-kgen-median > gpurun_out/bench_cfg4.log 2>&1
python bench.py --mode coarse --steps 300 --no-cpu-baseline > gpurun_out/bench_coarse.log 2>&1
python bench.py --mode coarse --config cfg3o --steps 300 --no-cpu-baseline > gpurun_out/bench_coarse_cfg3o.log 2>&1
python bench.py --mode absorb --steps 500 > gpurun_out/bench_absorb_cfg3o.log 2>&1
for f in gpurun_out/bench_*.log; do echo "$f $(tail -1 $f | cut -c1-120)"; done
