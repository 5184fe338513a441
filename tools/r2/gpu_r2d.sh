mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "csr or parity_s or extended or tiny or small_edges or vocab_shard or native_sharded_nccl or status or ignore or w_zero or accumulate or rmsnorm or split or host_input or native_dp_world1" > gpurun_out/r2d_tests.log 2>&1; echo tests $?; tail -5 gpurun_out/r2d_tests.log
timeout 600 python tools/bench_rmsnorm_lce.py > gpurun_out/r2d_rmsnorm.json 2> gpurun_out/r2d_rmsnorm.err; echo rms $?; cat gpurun_out/r2d_rmsnorm.json | head -c 1500; echo
timeout 600 python bench.py --steps 10 --warmup 3 --dist zipf --alpha 4 --no-cpu-baseline > gpurun_out/r2d_bench_zipf.json 2>/dev/null; echo zipf $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench.json 2>/dev/null; echo uni $?
python - <<'PY'
import json
for f in ['gpurun_out/r2d_bench_zipf.json','gpurun_out/r2d_bench.json']:
    d=json.load(open(f)); print(f, d['ms_per_step'], d['step_ms'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'])
PY
