mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke $?
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench $?
python -c "
import json
d=json.load(open('gpurun_out/r2a_bench.json')); print(d['ms_per_step'], d['frac_of_peak_burst'], d['roofline']['frac'], d['clocks'], d['e2e']['value'])
"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_tests.log 2>&1; echo tests $?; tail -3 gpurun_out/r2a_tests.log
