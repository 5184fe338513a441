export PYTHONUNBUFFERED=1
for r in 1 2; do for v in "" "--p2p-stats" "--p2p-stats --p2p-dx"; do
SLF_COMM_SMS_FORCE=1 timeout 600 python bench.py --module $v --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/px.json 2>/tmp/px.err || tail -3 /tmp/px.err
python -c "
import json
d=json.load(open('/tmp/px.json')); print(round(d['ms_per_step'],2), d['config']['comm'], d['clocks']['sm_mhz'])
"
done; done
