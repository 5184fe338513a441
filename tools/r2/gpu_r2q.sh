mkdir -p gpurun_out/r2q
export PYTHONUNBUFFERED=1
O=gpurun_out/r2q
for i in 1 2; do
SLF_INTERLEAVE=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/lpt$i.json 2>/dev/null
for L in 64 128 256; do
SLF_IL_SEG=$L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/il${L}_$i.json 2>/dev/null
done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2q/*.json')):
    try: d=json.load(open(f))
    except Exception as e: print(f,'ERR',e); continue
    k=d['kernels']; print(f, round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if v['ms_per_step']>0.5}, d['clocks']['sm_mhz'], d['clocks']['power_w_median'], round(d['roofline']['frac'],4), round(d['roofline'].get('frac_at_this_clock',0),4))
PY
for L in 64 128; do SLF_IL_SEG=$L timeout 300 python tools/unit_stats.py --what group --chunk 2 > $O/units_il$L.txt 2>&1; grep -E "cycles per K-block|clock" $O/units_il$L.txt; done
SLF_IL_SEG=128 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:lce_group -s 5 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu128.txt 2>&1; grep -E "duration|dram__bytes|tensor" $O/ncu128.txt
