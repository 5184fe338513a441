mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -4
for S in S R; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --schedule $S > gpurun_out/bench_r1g_$S.json 2> gpurun_out/bench_r1g_$S.err; tail -2 gpurun_out/bench_r1g_$S.err
done
python -c "
import json
for f in ['gpurun_out/bench_r1g_S.json','gpurun_out/bench_r1g_R.json']:
    try:
        d=json.load(open(f)); print(f, d['ms_per_step'], d['tflops'], d['frac_of_peak_burst'], d['clocks'], json.dumps(d['kernels']))
    except Exception as e: print(f, e)
"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 80 -c 80 --csv --log-file gpurun_out/launches_r1g_S.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --schedule S > /dev/null 2>&1; echo ncu $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lce_group -s 1 -c 2 -o gpurun_out/prof_r1g_S python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --schedule S > gpurun_out/ncu_full_S.log 2>&1; echo ncu2 $?
timeout 300 python tools/diag_s.py --schedule S
