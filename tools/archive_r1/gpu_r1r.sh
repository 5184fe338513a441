mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python bench.py --module --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mod_native.json 2> gpurun_out/bench_mod_native.err; echo native $?; tail -3 gpurun_out/bench_mod_native.err
timeout 600 python bench.py --module --comm torch --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mod_torch.json 2> gpurun_out/bench_mod_torch.err; echo torch $?
python -c "
import json
for f in ('native','torch'):
  d=json.load(open(f'gpurun_out/bench_mod_{f}.json')); print(f, d['ms_per_step'], d['config']['plan'], d['config'].get('comm'), d['memory']['frac_of_global_logits'], d['e2e'])
"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1r.json 2>gpurun_out/bench_ref_r1r.err; echo ref $?; cat gpurun_out/bench_ref_r1r.json
