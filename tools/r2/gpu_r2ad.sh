mkdir -p gpurun_out/r2ad
export PYTHONUNBUFFERED=1
O=gpurun_out/r2ad
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "llama_head or extended or small or edge or host or graph or rmsnorm" > $O/tests.log 2>&1; echo tests $?; tail -3 $O/tests.log
for i in 1 2 3; do
for e in 1 0; do
SLF_EARLY_MAINLOOP=$e timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/b_e${e}_$i.json 2>/dev/null; echo b $e $?
done; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2ad/b_*.json')):
    d=json.load(open(f)); k=d['kernels']; print(f, round(d['ms_per_step'],3), d['step_ms']['median'], round(k['gemm_stats']['ms_per_step'],3), round(k['gemm_group']['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['roofline']['frac'],4))
PY
