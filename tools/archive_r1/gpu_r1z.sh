mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for m3 in 1 0; do
for mn in 00 11; do echo "== debug mn=$mn MN3D=$m3"; SLF_MN3D=$m3 timeout 300 python tools/unit_stats.py --what debug --mn $mn 2>&1 | grep -E "debug GEMM|cycles per|wait full|rror"; done
echo "== group MN3D=$m3"; SLF_MN3D=$m3 timeout 300 python tools/unit_stats.py --what group --chunk 2 2>&1 | grep -E "cycles per|wait full|wait TMEM|slowest|rror"
done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1z.log 2>&1; echo pytest $?; tail -3 gpurun_out/pytest_gpu_r1z.log
for r in 1 2; do for m3 in 1 0; do
SLF_MN3D=$m3 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab3_$m3.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/ab3_$m3.json')); k=d['kernels']; print('MN3D=$m3', round(d['ms_per_step'],2), round(d['frac_of_peak_burst'],4), 'group', round(k['gemm_group']['ms_per_step'],2), round(k['gemm_group']['tflops']), 'stats', round(k['gemm_stats']['ms_per_step'],2), d['clocks']['sm_mhz'])
"
done; done
