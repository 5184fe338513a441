mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_train.py -m gpu -x -q -s > gpurun_out/r2f_tests.log 2>&1; echo tests $?; grep -E "train loop|passed|failed|Error" gpurun_out/r2f_tests.log | head
timeout 600 python tools/bench_rmsnorm_lce.py > gpurun_out/r2f_rmsnorm.json 2> gpurun_out/r2f_rmsnorm.err; echo rms $?; python -c "
import json; d=json.load(open('gpurun_out/r2f_rmsnorm.json')); print({k:d[k] for k in ['fused_ms_median','composed_ms_median','saved_ms_median','kernel_ms_per_step','extra_device_bytes']})"
timeout 900 python tools/bench_train_step.py > gpurun_out/r2f_train.json 2> gpurun_out/r2f_train.err; echo train $?; cat gpurun_out/r2f_train.json; tail -3 gpurun_out/r2f_train.err
