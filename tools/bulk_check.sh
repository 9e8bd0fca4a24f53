# A/B of the superposition's weight stream on cfg3 / cfg5: TMA-staged rows (default) vs
# per-thread 128-bit loads (--no-bulk-stream); device-timed bench lines
for v in "" "--no-bulk-stream"; do for c in cfg3 cfg5; do timeout 300 python bench.py --config $c $v --steps 100 --no-variants --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(\"$v\", \"$c\", round(d[\"ms_per_step\"],4), round(d[\"roofline\"][\"frac\"],4), d[\"clocks\"][\"sm_mhz\"])"; done; done
