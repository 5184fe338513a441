mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for C in qwen7b llama70b mistral123b; do
  for S in S R; do
    timeout 900 python bench.py --config $C --schedule $S --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r1t_${C}_${S}.json 2>/dev/null
    python -c "
import json
d=json.load(open('gpurun_out/bench_r1t_${C}_${S}.json')); print('$C', '$S', round(d['ms_per_step'],2), round(d['frac_of_peak_burst'],4), d['clocks']['sm_mhz'], round(d['memory']['frac_of_logits_per_gpu'],4))
"
  done
done
