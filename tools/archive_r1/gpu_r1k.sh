mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m "gpu and not slow" 2>&1 | tail -3
timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full|fwd only"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r1k.json 2> gpurun_out/bench_r1k.err; tail -2 gpurun_out/bench_r1k.err
python -c "
import json
d=json.load(open('gpurun_out/bench_r1k.json')); print(d['ms_per_step'], d['tflops'], d['frac_of_peak_burst'], d['clocks'], d['e2e'], json.dumps({k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()}))
"
