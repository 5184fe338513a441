mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nproc; free -g | head -2
timeout 2400 python -m pytest tests/test_gpu_heads.py "tests/test_gpu_parity.py::test_native_sharded_p2p_dx_uneven_shards" "tests/test_gpu_parity.py::test_native_sharded_callbacks" -m gpu -x -q -s --durations=20 > gpurun_out/r2b_tests.log 2>&1; echo tests $?; tail -40 gpurun_out/r2b_tests.log
