mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/bench_r1q.json 2> gpurun_out/bench_r1q.err; tail -2 gpurun_out/bench_r1q.err
python -c "
import json
d=json.load(open('gpurun_out/bench_r1q.json')); print(d['ms_per_step'], d['tflops'], d['frac_of_peak_burst'], d['roofline']['frac'], d['clocks'], d['e2e']['value'], d['cpu_baseline'])
"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 80 --csv --log-file gpurun_out/launches_r1q.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lce_group -s 4 -c 2 -o gpurun_out/prof_r1q python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:combine_transform -s 2 -c 1 -o gpurun_out/prof_r1q_ct python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu3 $?
for C in qwen7b llama70b mistral123b; do
timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r1q_$C.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/bench_r1q_$C.json')); print('$C', round(d['ms_per_step'],2), round(d['frac_of_peak_burst'],4), d['clocks']['sm_mhz'])
"
done
