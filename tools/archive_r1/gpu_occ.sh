python - <<'PY'
import ctypes, torch
torch.cuda.init()
l = ctypes.CDLL("paper_2603_16428_b200/libslf_lce.so")
f = l.slf_debug_max_active_clusters; f.argtypes=[ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
for c in (1,2,4,8,16):
    n = ctypes.c_int(0); r = f(c, ctypes.byref(n)); print("cluster", c, "rc", r, "max active clusters", n.value, "SMs", n.value*c)
PY
