export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_g8.log 2>&1; echo pytest $?; tail -2 gpurun_out/pytest_g8.log
for r in 1 2; do for m in 1 0; do
SLF_MN3D=$m timeout 600 python bench.py --module --emulate-shards 8 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/g8.json 2>/dev/null
python -c "
import json
d=json.load(open('/tmp/g8.json')); k=d['kernels']; print('MN3D=$m', round(d['ms_per_step'],3), 'group', round(k['gemm_group']['ms_per_step'],3), d['clocks']['sm_mhz'])
"
done; done
