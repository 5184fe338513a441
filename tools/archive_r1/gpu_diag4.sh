export PYTHONUNBUFFERED=1
for O in "4 0" "4 4" "6 8" "8 12"; do set -- $O; echo "OVH=$1 RMW=$2"; SLF_LPT_OVH=$1 SLF_LPT_RMW=$2 timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full"; done
timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full|fwd only"
