"""Host<->device copy rates on this box: pinned / pageable, H2D / D2H, at the
sizes the harness moves (1.2 MB = one NPB C vector), plus host memcpy rates
with 1..8 threads (numpy copies release the GIL)."""
import json
import threading
import time

import numpy as np
import torch


def rate(fn, nbytes, reps=50):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9


out = {}
for mb in (1.2, 16.0):
    n = int(mb * 1e6 / 8)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    hp = torch.empty(n, dtype=torch.float64).pin_memory()
    hg = torch.from_numpy(np.zeros(n))
    out[f"{mb}MB"] = {
        "h2d_pinned": rate(lambda: d.copy_(hp), n * 8),
        "d2h_pinned": rate(lambda: hp.copy_(d), n * 8),
        "h2d_pageable": rate(lambda: d.copy_(hg), n * 8),
        "d2h_pageable": rate(lambda: hg.copy_(d), n * 8),
    }
n = int(16e6 / 8)
src, dst = np.ones(n), np.zeros(n)
for T in (1, 2, 4, 8):
    parts = np.array_split(np.arange(n), T)
    bounds = [(p[0], p[-1] + 1) for p in parts]

    def work():
        ths = [threading.Thread(target=lambda a=a, b=b: np.copyto(dst[a:b], src[a:b])) for a, b in bounds]
        [t.start() for t in ths]
        [t.join() for t in ths]
    work()
    t = time.perf_counter()
    for _ in range(20):
        work()
    out[f"host_memcpy_{T}t_GBs"] = n * 8 * 20 / (time.perf_counter() - t) / 1e9
print(json.dumps(out, indent=1))
