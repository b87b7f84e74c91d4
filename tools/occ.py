import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_05215_b200 import _lib as L
p = torch.cuda.get_device_properties(0)
print("ctas/sm", L.lib().dz_sbmm_ctas_per_sm(), "smem/SM", p.shared_memory_per_multiprocessor, "optin", p.shared_memory_per_block_optin)
import ctypes as C
f = L.lib().dz_sbmm_diag
f.argtypes = [C.c_void_p]
v = (C.c_int * 8)()
f(v)
print("regs", v[0], "static smem", v[1], "dyn smem", v[2], "max threads", v[3], "local", v[4], "avail@2", v[5], "occ w carveout", v[6])
