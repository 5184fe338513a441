export PYTHONUNBUFFERED=1
O=gpurun_out/emu_r02
mkdir -p $O
for c in llama8b llama70b; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${c}_1.json 2>/dev/null; echo $c 1 $?
  for G in 2 4 8; do
    timeout 900 python bench.py --config $c --module --emulate-shards $G --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/${c}_$G.json 2>/dev/null; echo $c $G $?
  done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/emu_r02/*.json')):
    try: d=json.load(open(f))
    except Exception as e: print(f,'ERR',e); continue
    print(f, round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['config'].get('comm'))
PY
