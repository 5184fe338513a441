mkdir -p gpurun_out/r2l
export PYTHONUNBUFFERED=1
O=gpurun_out/r2l
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > $O/tests.log 2>&1; echo tests $?; tail -4 $O/tests.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/new$i.json 2>/dev/null
SLF_DEBUG_EPI=4096 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/oldstg$i.json 2>/dev/null
SLF_STAGING=4 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/stg4_$i.json 2>/dev/null
done
timeout 600 python bench.py --module --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/module.json 2>/dev/null; echo module $?
SLF_S_CLASSIC=1 timeout 600 python bench.py --module --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/module_classic.json 2>/dev/null; echo module2 $?
timeout 600 python bench.py --module --emulate-shards 8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/emu8.json 2>/dev/null; echo emu $?
SLF_S_CLASSIC=1 timeout 600 python bench.py --module --emulate-shards 8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/emu8_classic.json 2>/dev/null; echo emu2 $?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2l/*.json')):
    try: d=json.load(open(f))
    except Exception as e: print(f,'ERR',e); continue
    k=d['kernels']; print(f, round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if v['ms_per_step']>0.05}, d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))
PY
