mkdir -p gpurun_out/r2al
export PYTHONUNBUFFERED=1
O=gpurun_out/r2al
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/tests.log 2>&1; echo tests $?; tail -4 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -1 $O/smoke.log
for i in 1 2 3; do
SLF_INKERNEL_COMBINE=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_off_$i.json 2>/dev/null; echo b $?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_on_$i.json 2>/dev/null; echo n $?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2al/b_*.json')):
    d=json.load(open(f)); print(f, round(d['ms_per_step'],3), round(d['step_ms']['median'],3), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))
PY
