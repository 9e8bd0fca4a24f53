# profiles: the bench command's launch list (cold, serialised) and one `ncu --set full`
# capture each of the superposition (cfg3) and kgen (cfg3) kernels; summaries by tools/ncu_summary.py
set -x
python -c "import __graft_entry__ as g; g.build()"
B="python bench.py --steps 4 --warmup 3 --no-variants --no-checks --no-cpu-baseline --no-scaling-384"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B \
  > gpurun_out/launches_bench.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:superpose_bulk -s 3 -c 1 \
  -o gpurun_out/superpose_cfg3 -f $B > gpurun_out/ncu_sup.log 2>&1
echo sup_rc=$?
ncu --set full --clock-control none --import-source on -k regex:kgen -s 1 -c 1 \
  -o gpurun_out/kgen_cfg3 -f python tools/kgen_timing.py cfg3 2 > gpurun_out/ncu_kgen.log 2>&1
echo kgen_rc=$?
python tools/ncu_summary.py report gpurun_out/superpose_cfg3.ncu-rep gpurun_out/superpose_cfg3_ncu --config cfg3
python tools/ncu_summary.py report gpurun_out/kgen_cfg3.ncu-rep gpurun_out/kgen_cheb_cfg3_ncu --config cfg3
python tools/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/launches_bench_cfg3.txt
ls -la gpurun_out/
