export PYTHONUNBUFFERED=1
for D in 0 1 2 3; do echo "SLF_DEBUG_EPI=$D"; SLF_DEBUG_EPI=$D timeout 300 python tools/diag_s.py --schedule S 2>&1 | grep -E "full|dW only"; done
