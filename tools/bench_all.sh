# every BASELINE config and NEXT-row mode through bench.py, one JSON line each → gpurun_out/bench_<name>.json (copy the ones to keep into profiles/<round>_bench_<name>.json)
python -c "import __graft_entry__ as g; g.build()"
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name rc=$?"; }
run cfg1 --config cfg1 --steps 200 --warmup 10 --no-scaling-384
run cfg2 --config cfg2 --steps 200 --warmup 10
run cfg2_fp32 --config cfg2 --weights fp32 --steps 200 --warmup 10 --no-variants
run cfg5 --config cfg5 --steps 50 --warmup 5 --no-variants
run cfg3o --config cfg3o --steps 200 --warmup 10
run cfg3_mx8 --config cfg3 --weights mx8 --steps 200 --warmup 10 --no-scaling-384 --no-checks
run cfg3_dedup --config cfg3 --storage dedup --steps 200 --warmup 10 --no-checks
run coarse --mode coarse --steps 500 --warmup 20
run coarse_cfg3o --mode coarse --config cfg3o --steps 500 --warmup 20
run absorb --mode absorb --steps 300 --warmup 10
run absorb_mx8 --mode absorb --weights mx8 --steps 300 --warmup 10
