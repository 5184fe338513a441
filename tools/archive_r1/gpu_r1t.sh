mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python tools/bench_adam.py --config llama8b --steps 3 > gpurun_out/bench_adam_r1t.json 2> gpurun_out/bench_adam_r1t.err; echo adam $?; cat gpurun_out/bench_adam_r1t.json; tail -3 gpurun_out/bench_adam_r1t.err
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1t.log 2>&1; echo pytest $?; tail -3 gpurun_out/pytest_gpu_r1t.log
