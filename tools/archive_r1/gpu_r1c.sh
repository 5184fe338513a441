mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --schedule S > gpurun_out/bench_r1c_S.json 2> gpurun_out/bench_r1c_S.err; tail -2 gpurun_out/bench_r1c_S.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --schedule R > gpurun_out/bench_r1c_R.json 2> gpurun_out/bench_r1c_R.err; tail -2 gpurun_out/bench_r1c_R.err
python -c "
import json
for f in ['gpurun_out/bench_r1c_S.json','gpurun_out/bench_r1c_R.json']:
    try:
        d=json.load(open(f)); print(f, d['ms_per_step'], d['tflops'], d['frac_of_peak_burst'], d['clocks'], json.dumps(d['kernels']))
    except Exception as e: print(f, e)
"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and slow" 2>&1 | tail -8
