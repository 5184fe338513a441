mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for v in "" "--p2p-stats"; do
timeout 600 python bench.py --module $v --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mod$v.json 2> gpurun_out/bench_mod$v.err; echo rc $?; tail -2 gpurun_out/bench_mod$v.err
python -c "
import json
d=json.load(open('gpurun_out/bench_mod$v.json')); print('$v', d['ms_per_step'], d['config']['comm'], d['clocks']['sm_mhz'], d['e2e']['ms_per_step'])
"
done
