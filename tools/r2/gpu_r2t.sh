mkdir -p gpurun_out/r2t
export PYTHONUNBUFFERED=1
O=gpurun_out/r2t
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -m "gpu and not slow" -x -q > $O/tests.log 2>&1; echo tests $?; tail -2 $O/tests.log
for i in 1 2 3; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/cs8_$i.json 2>/dev/null
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2t/*.json')):
    d=json.load(open(f)); k=d['kernels']; print(f, round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if v['ms_per_step']>0.2}, d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))
PY
