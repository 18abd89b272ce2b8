"""Phase timestamps (clock64) of the standalone select kernel, sequence 0,
from a -DSKV_SELECT_TRACE build (SKV_LIB=build_var/libtrace.so)."""
import ctypes as C, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_17312_b200 import api
from paper_2403_17312_b200._lib import lib

for n in (128, 768, 1536, 4096):
    imp = torch.rand(16, n, device="cuda", dtype=torch.float64)
    for _ in range(3):
        api.swa_select(imp, n, 0.2)
    torch.cuda.synchronize()
    t = (C.c_longlong * 16)()
    lib().skv_debug_select_trace(t)
    print(f"n={n}: stage {t[1]-t[0]} | keys {t[2]-t[1]} | radix {t[10]-t[2]} ({t[8]} passes from bit {t[9]}) | compact {t[3]-t[10]} | total {t[3]-t[0]} cycles")
