python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
