mkdir -p gpurun_out/r2av
export PYTHONUNBUFFERED=1
O=gpurun_out/r2av
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke $?; tail -1 $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_heads.py -m gpu -q -x -k "llama_head or inkernel or mistral or qwen or extended" > $O/tests.log 2>&1; echo tests $?; tail -2 $O/tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2>/dev/null; echo bench $?; python -c "import json; d=json.load(open('$O/bench.json')); print(d['ms_per_step'], d['gpu_launches'], d['config']['plan'])"
