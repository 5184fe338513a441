export PYTHONUNBUFFERED=1
echo "base(TMA)"; timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full|dW only"
echo "LSU"; SLF_DEBUG_EPI=16 timeout 300 python tools/diag_s.py --schedule S --iters 8 2>&1 | grep -E "full|dW only"
echo "LSU parity"; SLF_DEBUG_EPI=16 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "tiny_parity or multichunk or shard_emulation_s" 2>&1 | tail -2
