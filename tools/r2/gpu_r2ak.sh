mkdir -p gpurun_out/r2ak
export PYTHONUNBUFFERED=1
O=gpurun_out/r2ak
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fallback or llama_head or small or edge" > $O/tests1.log 2>&1; echo tests1 $?; tail -3 $O/tests1.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heads.py tests/test_gpu_train.py -m gpu -q -k "not native" > $O/tests2.log 2>&1; echo tests2 $?; tail -3 $O/tests2.log
for i in 1 2 3 4; do
SLF_INKERNEL_COMBINE=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_off_$i.json 2>/dev/null; echo b $?
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_on_$i.json 2>/dev/null; echo n $?
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2ak/b_*.json')):
    d=json.load(open(f)); print(f, round(d['ms_per_step'],3), round(d['step_ms']['median'],3), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))
PY
