mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m "gpu" 2>&1 | tail -6
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r1l.json 2> gpurun_out/bench_r1l.err; tail -2 gpurun_out/bench_r1l.err
python -c "
import json
d=json.load(open('gpurun_out/bench_r1l.json')); print(d['ms_per_step'], d['tflops'], d['frac_of_peak_burst'], d['clocks'], d['e2e']['value'])
"
