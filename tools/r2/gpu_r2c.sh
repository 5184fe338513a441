mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "csr or parity_s or extended or tiny or small_edges or vocab_shard or native_sharded_nccl or status or ignore or w_zero or accumulate" > gpurun_out/r2c_tests.log 2>&1; echo tests $?; tail -5 gpurun_out/r2c_tests.log
for d in "uniform 1" "zipf 4"; do set -- $d
  timeout 300 python bench.py --steps 10 --warmup 3 --dist $1 --alpha $2 --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench_$1.json 2>/dev/null
  SLF_CSR_BRUTE=1 SLF_ONEHOT_SERIAL=1 timeout 300 python bench.py --steps 10 --warmup 3 --dist $1 --alpha $2 --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench_$1_old.json 2>/dev/null
done
for c in mistral123b llama70b; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --dist zipf --alpha 4 --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench_${c}_zipf.json 2>/dev/null
  SLF_CSR_BRUTE=1 SLF_ONEHOT_SERIAL=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --dist zipf --alpha 4 --no-cpu-baseline --no-e2e > gpurun_out/r2c_bench_${c}_zipf_old.json 2>/dev/null
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2c_bench_*.json')):
    try: d=json.load(open(f))
    except Exception as e: print(f, 'ERR', e); continue
    k=d['kernels']; print(f, round(d['ms_per_step'],3), 'csr', round(k.get('csr',{}).get('ms_per_step',0),4), 'onehot', round(k.get('onehot',{}).get('ms_per_step',0),4), 'median', round(d['step_ms']['median'],3), d['clocks']['sm_mhz'])
PY
