export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host_input" > gpurun_out/pytest_e2e.log 2>&1; echo pytest $?; tail -3 gpurun_out/pytest_e2e.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; echo bench $?; tail -2 gpurun_out/bench_e2e.err
python -c "
import json
d=json.load(open('gpurun_out/bench_e2e.json')); print(d['ms_per_step'], d['e2e'], d['clocks'])
"
