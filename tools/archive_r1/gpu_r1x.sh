mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for r in 1 2; do
for dbg in 0 1024; do
echo "== dbg=$dbg"
SLF_DEBUG_EPI=$dbg timeout 300 python tools/unit_stats.py --what group --chunk 2 2>&1 | tail -7
done
done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r1x.log 2>&1; echo pytest $?; tail -3 gpurun_out/pytest_gpu_r1x.log
