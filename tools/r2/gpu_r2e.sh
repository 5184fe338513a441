mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_parity.py -m gpu -x -q -s -k "train or upstream or graph or rmsnorm or autograd or split or accumulate or tiny" > gpurun_out/r2e_tests.log 2>&1; echo tests $?; grep -E "train loop|passed|failed|Error" gpurun_out/r2e_tests.log | head
timeout 600 python tools/bench_rmsnorm_lce.py > gpurun_out/r2e_rmsnorm.json 2> gpurun_out/r2e_rmsnorm.err; echo rms $?; python -c "
import json; d=json.load(open('gpurun_out/r2e_rmsnorm.json')); print({k:d[k] for k in ['fused_ms_median','composed_ms_median','saved_ms_median','rmsnorm_kernels','extra_device_bytes']})"
timeout 900 python tools/bench_train_step.py > gpurun_out/r2e_train.json 2> gpurun_out/r2e_train.err; echo train $?; cat gpurun_out/r2e_train.json; tail -3 gpurun_out/r2e_train.err
