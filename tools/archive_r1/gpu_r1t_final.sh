mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/bench_r1t.json 2> gpurun_out/bench_r1t.err; tail -2 gpurun_out/bench_r1t.err
python -c "
import json
d=json.load(open('gpurun_out/bench_r1t.json')); print(d['ms_per_step'], d['frac_of_peak_burst'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['energy'])
"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 80 --csv --log-file gpurun_out/launches_r1t.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lce_group -s 4 -c 2 -o gpurun_out/prof_r1t python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2 $?
