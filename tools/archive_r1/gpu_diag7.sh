export PYTHONUNBUFFERED=1
for G in 8 4 2 1 16; do echo "GROUP_M=$G"; SLF_GROUP_M=$G timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full|dW only"; done
