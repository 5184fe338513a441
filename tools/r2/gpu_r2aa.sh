mkdir -p gpurun_out/r2aa
export PYTHONUNBUFFERED=1
O=gpurun_out/r2aa
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > $O/tests.log 2>&1; echo tests $?; tail -20 $O/tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench $?
timeout 600 python bench.py --module --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/module.json 2>/dev/null; echo module $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2aa/*.json')):
    try: d=json.load(open(f))
    except Exception as e: print(f,'ERR',e); continue
    k=d['kernels']; print(f, round(d['ms_per_step'],3), d.get('frac_of_peak_burst'), (d.get('roofline') or {}).get('frac'), d['clocks']['sm_mhz'], (d.get('e2e') or {}).get('value'), {n: round(v['ms_per_step'],3) for n,v in k.items() if v['ms_per_step']>0.1})
PY
