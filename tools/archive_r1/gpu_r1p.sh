mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1p.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke_r1p.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1p.log 2>&1; echo pytest $?; tail -3 gpurun_out/pytest_gpu_r1p.log
timeout 900 python bench.py > gpurun_out/bench_r1p.json 2> gpurun_out/bench_r1p.err; tail -2 gpurun_out/bench_r1p.err
python -c "
import json
d=json.load(open('gpurun_out/bench_r1p.json')); print(d['ms_per_step'], d['tflops'], d['frac_of_peak_burst'], d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'])
"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1p.json 2>gpurun_out/bench_ref_r1p.err; echo ref $?; cat gpurun_out/bench_ref_r1p.json
