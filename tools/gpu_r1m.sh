mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x 2>&1 | grep -v "^\s*$" | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r1m.json 2> gpurun_out/bench_r1m.err; tail -2 gpurun_out/bench_r1m.err
python -c "
import json
d=json.load(open('gpurun_out/bench_r1m.json')); print(d['ms_per_step'], d['tflops'], d['frac_of_peak_burst'], d['clocks'], d['e2e']['ms_per_step'], sum(k['ms_per_step'] for k in d['kernels'].values()))
"
