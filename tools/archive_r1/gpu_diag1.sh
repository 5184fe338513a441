export PYTHONUNBUFFERED=1
timeout 300 python tools/diag_s.py --schedule S
timeout 300 python tools/diag_s.py --schedule S --budget-mult 2
timeout 300 python tools/diag_s.py --schedule R
