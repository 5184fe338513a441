mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x 2>&1 | grep -v "^\s*$" | tail -3
for i in 1 2; do
echo "mixed (default)"; timeout 300 python tools/diag_s.py 2>&1 | sed -n 2,2p
echo "all 4 bufs"; SLF_STAGING=4 timeout 300 python tools/diag_s.py 2>&1 | sed -n 2,2p
done
