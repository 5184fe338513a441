mkdir -p gpurun_out/r2r
export PYTHONUNBUFFERED=1
O=gpurun_out/r2r
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?
timeout 2400 python -m pytest tests -m gpu -q --durations=5 > $O/tests.log 2>&1; echo tests $?; tail -12 $O/tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench $?
python -c "
import json; d=json.load(open('$O/bench.json')); print(d['ms_per_step'], d['value'], d['frac_of_peak_burst'], d['roofline'], d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'])"
