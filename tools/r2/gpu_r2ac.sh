mkdir -p gpurun_out/r2ac
export PYTHONUNBUFFERED=1
O=gpurun_out/r2ac
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heads.py -m gpu -q -k "sharded or shard or dp_ or module" > $O/tests.log 2>&1; echo tests $?; tail -3 $O/tests.log
for i in 1 2; do
timeout 600 python bench.py --module --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/module_$i.json 2>/dev/null; echo module $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/fused_$i.json 2>/dev/null; echo fused $?
done
SLF_SHARD_PART=region timeout 600 python bench.py --module --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/module_region.json 2>/dev/null; echo region $?
timeout 600 python bench.py --module --emulate-shards 8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/emu8.json 2>/dev/null; echo emu $?
timeout 600 python bench.py --module --emulate-shards 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/emu2.json 2>/dev/null; echo emu2 $?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2ac/*.json')):
    try: d=json.load(open(f))
    except Exception as e: print(f,'ERR',e); continue
    k=d['kernels']; print(f, round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if v['ms_per_step']>0.1}, d['clocks']['sm_mhz'], d['config']['plan'][:200])
PY
