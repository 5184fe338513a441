export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "native_sharded or no_device_alloc" > gpurun_out/pytest_r1rs.log 2>&1; echo pytest $?; tail -3 gpurun_out/pytest_r1rs.log
for k in 0 4 8; do
SLF_COMM_SMS_FORCE=1 timeout 900 python bench.py --module --comm-sms $k --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/rs_$k.json 2>/dev/null
python -c "
import json
d=json.load(open('/tmp/rs_$k.json')); print('reserve $k', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])
"
done
