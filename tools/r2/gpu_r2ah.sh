mkdir -p gpurun_out/r2ah
export PYTHONUNBUFFERED=1
O=gpurun_out/r2ah
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -m gpu -q -k "llama_head or extended or small or edge or host or graph or rmsnorm or all_chunk_kinds or train" > $O/tests.log 2>&1; echo tests $?; tail -3 $O/tests.log
