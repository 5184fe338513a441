mkdir -p gpurun_out/r2am
export PYTHONUNBUFFERED=1
O=gpurun_out/r2am
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "inkernel_combine or interleaved" > $O/tests.log 2>&1; echo tests $?; tail -3 $O/tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lce_group -s 4 -c 2 -o $O/prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2 $?
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2am/bench.json')); print(d['ms_per_step'], d['step_ms'], d['clocks']['sm_mhz'], d['roofline']['frac'], d['frac_of_peak_burst'], (d.get('e2e') or {}).get('value'))
PY
