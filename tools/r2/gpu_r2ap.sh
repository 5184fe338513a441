mkdir -p gpurun_out/r2ap
export PYTHONUNBUFFERED=1
O=gpurun_out/r2ap
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench $?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo ref $?
timeout 600 python bench.py --dist zipf --alpha 4 --no-cpu-baseline > $O/bench_zipf.json 2>/dev/null; echo zipf $?
timeout 600 python bench.py --schedule R --no-cpu-baseline --no-e2e > $O/bench_R.json 2>/dev/null; echo R $?
timeout 600 python bench.py --module --no-cpu-baseline --no-e2e > $O/bench_module.json 2>/dev/null; echo module $?
for c in qwen7b llama70b mistral123b; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2>/dev/null; echo $c $?; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lce_group -s 4 -c 2 -o $O/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2 $?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2ap/bench*.json')):
    try: d=json.load(open(f))
    except Exception as e: print(f,'ERR',e); continue
    print(f, round(d.get('ms_per_step',0),3), d.get('value'), d.get('frac_of_peak_burst'), (d.get('roofline') or {}).get('frac'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('e2e') or {}).get('value'), (d.get('step_ms') or {}).get('median'))
PY
