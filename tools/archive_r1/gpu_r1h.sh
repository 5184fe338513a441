mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -3
for S in S R; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --schedule $S > gpurun_out/bench_r1h_$S.json 2> gpurun_out/bench_r1h_$S.err; tail -2 gpurun_out/bench_r1h_$S.err
done
python -c "
import json
for f in ['gpurun_out/bench_r1h_S.json','gpurun_out/bench_r1h_R.json']:
    try:
        d=json.load(open(f)); print(f, d['ms_per_step'], d['tflops'], d['frac_of_peak_burst'], d['clocks'], json.dumps({k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()}))
    except Exception as e: print(f, e)
"
