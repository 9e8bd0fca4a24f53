# MX8 superposition at cfg3: parity, then stages per CTA A/B (FDIRW_MX8_STAGES)
timeout 900 python -m pytest tests/test_gpu_mx8.py -x -q 2>&1 | tail -3
for v in "" "FDIRW_MX8_STAGES=2" "FDIRW_MX8_STAGES=3"; do
  echo "== $v"
  env $v timeout 300 python bench.py --weights mx8 --no-variants --no-cpu-baseline --steps 200 --e2e-steps 5 --no-kgen-median 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['read_ceiling']['frac'], d['mass_rel_err'])"
done
