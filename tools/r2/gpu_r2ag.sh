mkdir -p gpurun_out/r2ag
export PYTHONUNBUFFERED=1
O=gpurun_out/r2ag
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -m gpu -q -x -k "llama_head or extended or small or edge or host or graph or rmsnorm or all_chunk_kinds or train" > $O/tests.log 2>&1; echo tests $?; tail -3 $O/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -2 $O/smoke.log
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/b_$i.json 2>/dev/null; echo b $?; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2ag/b_*.json')):
    d=json.load(open(f)); print(f, round(d['ms_per_step'],3), d['step_ms']['median'], d['clocks']['sm_mhz'], round(d['roofline']['frac'],4), round(d['frac_of_peak_burst'],4))
PY
