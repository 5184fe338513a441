mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for xt in 1 0; do echo "== group XT=$xt"; SLF_XT=$xt timeout 300 python tools/unit_stats.py --what group --chunk 2 2>&1 | grep -E "cycles per|wait full|slowest|rror"; done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1zb.log 2>&1; echo pytest $?; tail -3 gpurun_out/pytest_gpu_r1zb.log
for r in 1 2; do for xt in 1 0; do
SLF_XT=$xt timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abx_$xt.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/abx_$xt.json')); k=d['kernels']; print('XT=$xt', round(d['ms_per_step'],2), round(d['frac_of_peak_burst'],4), 'group', round(k['gemm_group']['ms_per_step'],2), round(k['gemm_group']['tflops']), 'stats', round(k['gemm_stats']['ms_per_step'],2), 'tr', k.get('transpose',{}).get('ms_per_step'), d['clocks']['sm_mhz'])
"
done; done
