mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for G in 2 4 8; do
timeout 900 python bench.py --config llama70b --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --module --emulate-shards $G > gpurun_out/bench_em70.json 2> gpurun_out/bench_em70.err; echo "G=$G rc=$?"
python -c "
import json
d=json.loads(open('gpurun_out/bench_em70.json').read()); print(round(d['ms_per_step'],2), d['config']['V_per_gpu'], d['config']['plan'], d['memory']['frac_of_global_logits'], d['clocks']['sm_mhz'])
"
done
timeout 900 python bench.py --config llama70b --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_70.json 2>/dev/null; python -c "
import json
d=json.loads(open('gpurun_out/bench_70.json').read()); print('fused g=1', round(d['ms_per_step'],2), d['frac_of_peak_burst'], d['config']['plan'], d['clocks']['sm_mhz'])
"
