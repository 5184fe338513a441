export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m "gpu and not slow" 2>&1 | tail -2
echo "TMA stash"; timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full|fwd only"
echo "thread stash"; SLF_DEBUG_EPI=64 timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full|fwd only"
