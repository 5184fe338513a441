export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/emu2
for C in llama8b llama70b; do for G in 2 4 8; do
timeout 900 python bench.py --config $C --module --emulate-shards $G --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/emu2/${C}_${G}_native.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/emu2/${C}_${G}_native.json')); print('$C G=$G', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])
"
done; done
for C in llama8b llama70b; do
timeout 900 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/emu2/${C}_1.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/emu2/${C}_1.json')); print('$C G=1', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])
"
done
