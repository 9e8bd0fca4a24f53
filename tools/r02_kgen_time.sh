python -c "import __graft_entry__ as g; g.build()"
python tools/kgen_timing.py cfg3 3
python tools/kgen_timing.py cfg5 3
timeout 900 python -m pytest tests -q -m gpu -x -k "kgen or dedup or cfg1 or edge or cfg5" 2>&1 | tail -3
