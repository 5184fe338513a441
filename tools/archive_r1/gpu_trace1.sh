export PYTHONUNBUFFERED=1
timeout 300 python tools/trace_tiles.py --chunk 2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m "gpu" -k "rmsnorm" 2>&1 | tail -3
