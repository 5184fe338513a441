mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/r2j_tests.log 2>&1; echo tests $?; tail -4 gpurun_out/r2j_tests.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_t$i.json 2>/dev/null
SLF_XS_T=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2j_bench_r$i.json 2>/dev/null
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2j_bench_*.json')):
    try: d=json.load(open(f))
    except Exception as e: print(f,'ERR',e); continue
    k=d['kernels']; print(f, round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items()}, d['clocks']['sm_mhz'], d['clocks']['power_w_median'], round(d['roofline']['frac'],4))
PY
