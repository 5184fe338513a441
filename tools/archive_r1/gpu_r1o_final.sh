mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/bench_r1o.json 2> gpurun_out/bench_r1o.err; tail -2 gpurun_out/bench_r1o.err
python -c "
import json
d=json.load(open('gpurun_out/bench_r1o.json')); print(d['ms_per_step'], d['tflops'], d['frac_of_peak_burst'], d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'])
"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 80 --csv --log-file gpurun_out/launches_r1o.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lce_group -s 4 -c 2 -o gpurun_out/prof_r1o python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:combine_transform -s 2 -c 1 -o gpurun_out/prof_r1o_ct python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu3 $?
