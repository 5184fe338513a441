mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
SLF_DW_ACC=3 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" -x 2>&1 | grep -v "^\s*$" | tail -1
SLF_DW_ACC=3 timeout 600 python tools/dw_acc_error.py
for i in 1 2; do
echo acc2; timeout 300 python tools/diag_s.py --iters 10 2>&1 | sed -n 2,4p
echo acc3; SLF_DW_ACC=3 timeout 300 python tools/diag_s.py --iters 10 2>&1 | sed -n 2,4p
done
