mkdir -p gpurun_out/r2au
export PYTHONUNBUFFERED=1
O=gpurun_out/r2au
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/tests.log 2>&1; echo tests $?; tail -2 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench $?
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2au/bench.json')); print(d['ms_per_step'], d['step_ms']['median'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['frac_of_peak_burst'], d['e2e']['value'], d['cpu_baseline']['value'])
PY
