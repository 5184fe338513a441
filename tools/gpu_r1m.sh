mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for G in 2 4 8; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --module --emulate-shards $G > gpurun_out/bench_em.json 2> gpurun_out/bench_em.err; echo "G=$G rc=$?"; tail -2 gpurun_out/bench_em.err | cut -c1-200
python -c "
import json
d=json.loads(open('gpurun_out/bench_em.json').read()); print(round(d['ms_per_step'],3), d['config']['V_per_gpu'], d['config']['plan'], {k: round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['memory']['frac_of_global_logits'])
"
done
