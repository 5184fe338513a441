mkdir -p gpurun_out/r2z
export PYTHONUNBUFFERED=1
O=gpurun_out/r2z
for ovh in 2 3; do
SLF_LPT_OVH=$ovh timeout 300 python tools/unit_stats.py --what group --chunk 2 > $O/units_ovh$ovh.txt 2>&1; echo ovh $ovh; tail -6 $O/units_ovh$ovh.txt
done
for i in 1 2; do for ovh in 4 3 2; do
SLF_LPT_OVH=$ovh timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_ovh${ovh}_$i.json 2>/dev/null
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2z/b_*.json')):
    d=json.load(open(f)); k=d['kernels']; print(f, round(d['ms_per_step'],3), round(k['gemm_group']['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))
PY
