python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 600 python tools/ab_fit.py --trees 100 --rounds 3 -- "" "LLMP_HIST2=5" "LLMP_HIST2=1"
