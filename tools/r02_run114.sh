python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
