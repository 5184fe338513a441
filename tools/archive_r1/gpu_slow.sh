export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests/test_gpu_parity.py -q -m "gpu and slow" 2>&1 | tail -5
