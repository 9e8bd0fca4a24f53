# e2e A/B: fdirw_step_host pipelined (default) vs the plain form (FDIRW_STEP_HOST_CHUNKS=1)
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -q -m gpu -x -k "step_host or profile_phases or canary" 2>&1 | tail -2
B="python bench.py --steps 20 --warmup 5 --no-variants --no-checks --no-cpu-baseline --no-scaling-384"
for n in 0 1 8 12 16; do
  FDIRW_STEP_HOST_CHUNKS=$n $B > gpurun_out/e2e_$n.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e2e_$n.json')); print('chunks=$n', 'value %.4g' % d['value'], 'e2e %.4g' % d['e2e']['value'], 'ratio %.3f' % (d['e2e']['value']/d['value']))"
done
