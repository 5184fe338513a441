mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for i in 1 2; do
echo base; timeout 300 python tools/diag_s.py --iters 10 2>&1 | sed -n 2,2p
echo mid; SLF_LPT_ORDER=mid timeout 300 python tools/diag_s.py --iters 10 2>&1 | sed -n 2,2p
done
