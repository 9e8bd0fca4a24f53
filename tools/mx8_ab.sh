# MX8 + N4 mixed launch at cfg3: stages per CTA A/B (FDIRW_MX8_STAGES: 3 = 2 CTAs/SM, 2 = 3 CTAs/SM)
for v in "" "FDIRW_MX8_STAGES=2" "FDIRW_MX8_STAGES=3"; do
  echo "== $v"
  env $v timeout 300 python bench.py --weights mx8 --storage dedup --no-variants --no-cpu-baseline --steps 300 --e2e-steps 5 --no-kgen-median 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
