python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
LLMP_HIST2=7 python bench.py > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
python bench.py > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
