export PYTHONUNBUFFERED=1
echo "base"; timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "dW only"
echo "store-only"; SLF_DEBUG_DW_NO_RMW=1 timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "dW only"
echo "no-load no-store"; SLF_DEBUG_DW_NO_RMW=1 SLF_DEBUG_EPI=8 timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "dW only"
echo "rmw-load no-store"; SLF_DEBUG_EPI=8 timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "dW only"
