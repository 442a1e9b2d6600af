"""Does mprotect work on torch pinned host memory? (diagnostic)"""
import ctypes
import ctypes.util
import numpy as np
import torch

libc = ctypes.CDLL(ctypes.util.find_library("c"), use_errno=True)
libc.mprotect.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
t = torch.zeros(150000, dtype=torch.float64, pin_memory=True)
a = t.numpy()
base = a.ctypes.data
page = 4096
lo = (base + page - 1) & ~(page - 1)
rc = libc.mprotect(lo, page * 4, 1)  # PROT_READ
print("pinned: addr%4096 =", base % 4096, "mprotect rc", rc, "errno", ctypes.get_errno())
rc = libc.mprotect(lo, page * 4, 3)
b = np.zeros(150000)
base = b.ctypes.data
lo = (base + page - 1) & ~(page - 1)
rc = libc.mprotect(lo, page * 4, 1)
print("pageable: mprotect rc", rc, "errno", ctypes.get_errno())
libc.mprotect(lo, page * 4, 3)
