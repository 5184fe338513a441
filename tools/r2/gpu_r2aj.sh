mkdir -p gpurun_out/r2aj
export PYTHONUNBUFFERED=1
O=gpurun_out/r2aj
# exposed cost of one combine launch per chunk: SLF_DEBUG_CT2=1 issues it twice (same outputs)
for i in 1 2 3 4; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_base_$i.json 2>/dev/null; echo b $?
SLF_DEBUG_CT2=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_ct2_$i.json 2>/dev/null; echo n $?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2aj/b_*.json')):
    d=json.load(open(f)); print(f, round(d['ms_per_step'],3), round(d['step_ms']['median'],3), d['clocks']['sm_mhz'])
PY
