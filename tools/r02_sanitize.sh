python -c "import __graft_entry__ as g; g.build()"
bash tools/sanitize_all.sh
