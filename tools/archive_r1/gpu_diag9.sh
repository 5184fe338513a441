export PYTHONUNBUFFERED=1
echo "base"; timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "fwd only"
echo "no stash stores"; SLF_DEBUG_EPI=32 timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "fwd only"
echo "R"; timeout 300 python tools/diag_s.py --schedule R --iters 8 2>&1 | grep -E "fwd only"
