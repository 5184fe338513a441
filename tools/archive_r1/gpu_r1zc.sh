export PYTHONUNBUFFERED=1
for r in 1 2 3 4 5; do for xt in 1 0; do
SLF_XT=$xt timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/abx_$xt.json 2>/dev/null
python -c "
import json
d=json.load(open('/tmp/abx_$xt.json')); k=d['kernels']; print('XT=$xt', round(d['ms_per_step'],3), 'group', round(k['gemm_group']['ms_per_step'],3), d['clocks']['sm_mhz'])
"
done; done
