mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_end.log 2>&1; echo smoke $?; tail -1 gpurun_out/smoke_end.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_end.log 2>&1; echo pytest $?; tail -2 gpurun_out/pytest_gpu_end.log
timeout 900 python bench.py > gpurun_out/bench_end.json 2> gpurun_out/bench_end.err; echo bench $?; tail -2 gpurun_out/bench_end.err
python -c "
import json
d=json.load(open('gpurun_out/bench_end.json')); print(d['ms_per_step'], d['tflops'], d['tflops_executed'], d['frac_of_peak_burst'], d['roofline'], d['clocks'], d['e2e'], d['cpu_baseline']['value'], d['gpu_launches'], d['memory'])
"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_end.json 2>gpurun_out/bench_ref_end.err; echo ref $?; cat gpurun_out/bench_ref_end.json | cut -c1-300
