export PYTHONUNBUFFERED=1
echo "order=first"; timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full"
echo "order=mid"; SLF_LPT_ORDER=mid timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full"
