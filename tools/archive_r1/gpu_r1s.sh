mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_layer_adam.py -x -q > gpurun_out/pytest_adam_r1s.log 2>&1; echo pytest $?; tail -5 gpurun_out/pytest_adam_r1s.log
lscpu | grep -E "Model name|^CPU\(s\)|Thread|NUMA node\(s\)" > gpurun_out/lscpu_r1s.txt; cat gpurun_out/lscpu_r1s.txt; free -g | head -2
timeout 900 python tools/bench_adam.py --config llama8b --steps 3 > gpurun_out/bench_adam_r1s.json 2> gpurun_out/bench_adam_r1s.err; echo adam $?; cat gpurun_out/bench_adam_r1s.json; tail -3 gpurun_out/bench_adam_r1s.err
