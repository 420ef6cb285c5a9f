set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "" "LLMP_PAIRED=1" "LLMP_PDL=0"; do
  env $v timeout 900 python bench.py --no-wg --no-cv --no-c5 --no-rf --no-cpu-baseline --no-e2e > gpurun_out/ab_$(echo $v | tr '=' '_').json 2>/dev/null
  python -c "import json,sys; j=json.load(open('gpurun_out/ab_$(echo $v | tr '=' '_').json')); print('$v', j['value']/1e9, j['fit']['ms_per_step'])"
done
