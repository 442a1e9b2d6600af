import time, sys
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2001_07938_b200 import _native as N
from paper_2001_07938_b200 import harness as H
N.check(N.lib().b200_init(0))
n = 150000
H.set_writeback("lazy")
a = H.page_aligned(n); b = H.page_aligned(n)
a[:] = 1.0; b[:] = 2.0
for _ in range(50): H.dotproduct(n, a, b)
t = time.perf_counter()
for _ in range(2000): H.dotproduct(n, a, b)
dt = (time.perf_counter() - t) / 2000
print("dot round trip (clean inputs, device mirrors): %.1f us" % (dt * 1e6))
y = H.page_aligned(n)
for _ in range(50): H.axpy(n, y, 0.5, a)
t = time.perf_counter()
for _ in range(2000): H.axpy(n, y, 0.5, a)
print("axpy call (lazy output): %.1f us" % ((time.perf_counter() - t) / 2000 * 1e6))
t = time.perf_counter()
for _ in range(1000):
    H.axpy(n, y, 0.5, a); H.dotproduct(n, y, y)
print("axpy+dot: %.1f us" % ((time.perf_counter() - t) / 1000 * 1e6))
