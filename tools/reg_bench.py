"""Time cudaHostRegister of hytgen (THP-backed) arrays with and without the
ReadOnly flag (load path of hyt_load_csr)."""
import ctypes, time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import hytgen
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
rt.cudaHostUnregister.argtypes = [ctypes.c_void_p]
for flags, name in ((2, "Mapped"), (2 | 8, "Mapped|ReadOnly")):
    a = hytgen.aligned_empty(2 << 30, np.uint32)     # 8 GB
    a[::1024] = 1
    t = time.time()
    rc = rt.cudaHostRegister(a.ctypes.data, a.nbytes, flags)
    t1 = time.time()
    rt.cudaHostUnregister(a.ctypes.data)
    t2 = time.time()
    print(f"{name}: register 8 GB {t1 - t:.3f}s rc={rc}, unregister {t2 - t1:.3f}s", flush=True)
    del a
