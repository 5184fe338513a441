mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/r2h_tests.log 2>&1; echo tests $?; tail -4 gpurun_out/r2h_tests.log
timeout 1500 python -m pytest tests -m "gpu and slow" -x -q -s -k "reduced_n or rmsnorm or llama8b" > gpurun_out/r2h_slow.log 2>&1; echo slow $?; grep -E "err|passed|failed" gpurun_out/r2h_slow.log | tail -12
