mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python tools/trace_tiles.py --chunk 2 2>&1 | tail -18
timeout 300 python tools/trace_tiles.py --chunk 14 2>&1 | tail -18
timeout 300 python tools/trace_tiles.py --chunk 2 --stats 2>&1 | tail -8
