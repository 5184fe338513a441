mkdir -p gpurun_out/r2ao
export PYTHONUNBUFFERED=1
O=gpurun_out/r2ao
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/tests.log 2>&1; echo tests $?; tail -3 $O/tests.log
for i in 1 2 3; do
SLF_S_REF_EXT=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_off_$i.json 2>/dev/null; echo b $?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_on_$i.json 2>/dev/null; echo n $?
done
for i in 1 2; do
SLF_S_REF_EXT=0 timeout 900 python bench.py --config llama70b --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/b70_off_$i.json 2>/dev/null; echo b70 $?
timeout 900 python bench.py --config llama70b --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/b70_on_$i.json 2>/dev/null; echo n70 $?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2ao/b*.json')):
    d=json.load(open(f)); print(f, round(d['ms_per_step'],3), round(d['step_ms']['median'],3), d['clocks']['sm_mhz'], d['config']['plan'][:90])
PY
