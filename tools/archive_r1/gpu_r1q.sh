mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "native_sharded" > gpurun_out/pytest_native_r1q.log 2>&1; echo pytest $?; tail -30 gpurun_out/pytest_native_r1q.log
