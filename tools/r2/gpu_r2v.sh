mkdir -p gpurun_out/r2v
export PYTHONUNBUFFERED=1
O=gpurun_out/r2v
timeout 600 python tools/bench_rmsnorm_lce.py --pairs 6 > $O/rmsnorm.json 2> $O/rmsnorm.err; echo rms $?; python -c "
import json; d=json.load(open('$O/rmsnorm.json')); print({k:d[k] for k in ['fused_ms_median','composed_ms_median','saved_ms_median','kernel_ms_per_step','extra_device_bytes']})"
timeout 900 python tools/bench_train_step.py > $O/train.json 2> $O/train.err; echo train $?; cat $O/train.json
