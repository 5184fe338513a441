mkdir -p gpurun_out/r2at
export PYTHONUNBUFFERED=1
O=gpurun_out/r2at
timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sharded or shard or dp_" > $O/tests.log 2>&1; echo tests $?; tail -2 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -1 $O/smoke.log
for i in 1 2 3; do
timeout 600 python bench.py --module --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/module_$i.json 2>/dev/null; echo module $?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/fused_$i.json 2>/dev/null; echo fused $?
done
timeout 600 python bench.py --module --emulate-shards 8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/emu8.json 2>/dev/null; echo emu8 $?
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2at/*.json')):
    d=json.load(open(f)); print(f, round(d['ms_per_step'],3), round(d['step_ms']['median'],3), d['clocks']['sm_mhz'])
PY
