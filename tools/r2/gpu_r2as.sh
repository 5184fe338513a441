mkdir -p gpurun_out/r2as
export PYTHONUNBUFFERED=1
O=gpurun_out/r2as
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "all_chunk_kinds or partial_placement" > $O/tests.log 2>&1; echo tests $?; tail -2 $O/tests.log
