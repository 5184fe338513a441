mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
echo base; timeout 300 python tools/diag_s.py --iters 10 2>&1 | sed -n 2,4p
echo nostore; SLF_DEBUG_EPI=256 timeout 300 python tools/diag_s.py --iters 10 2>&1 | sed -n 2,4p
done
SLF_DEBUG_EPI=256 timeout 300 python tools/unit_stats.py --what group --chunk 12 2>&1 | grep -v slowest | grep -v fastest
