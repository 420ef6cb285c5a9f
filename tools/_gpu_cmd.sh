python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python tools/ab_fit.py --trees 500 --reps 3 --rounds 2 -- "" "LLMP_HIST2=7"
