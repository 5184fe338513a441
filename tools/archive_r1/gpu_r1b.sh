mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 120 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" 2>&1 | tail -8
SLF_CTA_GROUP=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m "gpu and not slow" -k "gemm_core or tiny" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; tail -2 gpurun_out/bench_r1b.err
cat gpurun_out/bench_r1b.json
