mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests/ -q -m "gpu and not slow" -x 2>&1 | grep -v "^\s*$" | tail -2
