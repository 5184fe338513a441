mkdir -p gpurun_out/r2p
export PYTHONUNBUFFERED=1
O=gpurun_out/r2p
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > $O/tests.log 2>&1; echo tests $?; tail -4 $O/tests.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/il$i.json 2>/dev/null
SLF_INTERLEAVE=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/lpt$i.json 2>/dev/null
SLF_IL_SEG=32 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/il32_$i.json 2>/dev/null
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2p/*.json')):
    try: d=json.load(open(f))
    except Exception as e: print(f,'ERR',e); continue
    k=d['kernels']; print(f, round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if v['ms_per_step']>0.05}, d['clocks']['sm_mhz'], d['clocks']['power_w_median'], round(d['roofline']['frac'],4), round(d['roofline'].get('frac_at_this_clock',0),4))
PY
timeout 300 python tools/unit_stats.py --what group --chunk 2 > $O/units_group.txt 2>&1; tail -12 $O/units_group.txt
timeout 600 ncu --set full --clock-control none -k regex:lce_group -s 5 -c 1 -o $O/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
