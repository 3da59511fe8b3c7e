timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^\s*$" | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python tools/regions_time.py 2>&1 | tail -2
