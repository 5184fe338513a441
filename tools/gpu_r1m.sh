mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 300 python tools/diag_s.py --schedule S 2>&1 | tail -6
SLF_S_NO_EXT=1 timeout 300 python tools/diag_s.py --schedule S 2>&1 | tail -6
timeout 300 python tools/diag_s.py --schedule S 2>&1 | tail -6
