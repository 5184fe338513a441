mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for mn in 00 01 10 11; do echo "== debug mn=$mn"; timeout 300 python tools/unit_stats.py --what debug --mn $mn 2>&1 | grep -E "debug GEMM|cycles per|wait full|wait TMEM"; done
for dbg in 0 2048; do echo "== group dbg=$dbg"; SLF_DEBUG_EPI=$dbg timeout 300 python tools/unit_stats.py --what group --chunk 2 2>&1 | grep -E "cycles per|wait full|wait TMEM|slowest"; done
