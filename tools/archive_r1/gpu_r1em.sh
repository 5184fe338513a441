export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/emu
for C in llama8b llama70b; do for G in 2 4 8; do for cm in native torch; do
timeout 900 python bench.py --config $C --module --emulate-shards $G --comm $cm --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/emu/${C}_${G}_${cm}.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/emu/${C}_${G}_${cm}.json')); print('$C G=$G $cm', round(d['ms_per_step'],2), d['config']['plan'][:90], d['clocks']['sm_mhz'], round(d['memory']['frac_of_global_logits'],4))
"
done; done; done
