mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for r in 1 2; do
for dbg in 0 1024; do
SLF_DEBUG_EPI=$dbg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$dbg.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/ab_$dbg.json')); k=d['kernels']; print('dbg=$dbg', round(d['ms_per_step'],2), round(d['frac_of_peak_burst'],4), 'group', round(k['gemm_group']['ms_per_step'],2), round(k['gemm_group']['tflops']), 'stats', round(k['gemm_stats']['ms_per_step'],2), d['clocks']['sm_mhz'])
"
done
done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1w.log 2>&1; echo pytest $?; tail -3 gpurun_out/pytest_gpu_r1w.log
