"""EP curve (100 return periods) at 1M trials: wall time per call, device and host YLT."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1308_2066_b200.risk import ep_curve, order_stats
rng = np.random.default_rng(5)
x = np.minimum(rng.lognormal(8.0, 2.0, 1_000_000), 66_000.0)
d = torch.from_numpy(x).cuda()
rps = np.unique(np.concatenate([np.geomspace(1.01, 1e6, 97), [2.0, 10.0, 1e6]]))
for name, src in (("device", d), ("host", x)):
    for _ in range(5):
        ep_curve(src, rps)
    torch.cuda.synchronize()
    t = []
    for _ in range(50):
        t0 = time.perf_counter(); ep_curve(src, rps); t.append(time.perf_counter() - t0)
    print(name, "ep_curve 100 points: median %.3f ms, min %.3f ms" % (np.median(t) * 1e3, min(t) * 1e3))
t = []
for _ in range(50):
    t0 = time.perf_counter(); order_stats(d, [10, 50, 100, 250]); t.append(time.perf_counter() - t0)
print("order_stats 4 rps device: median %.3f ms" % (np.median(t) * 1e3))
# device components: torch's own sort of the same 1M float64 (CUB segmented/radix), for scale
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    torch.sort(d)
e[0].record()
for _ in range(20):
    torch.sort(d)
e[1].record(); torch.cuda.synchronize()
print("torch.sort 1M float64: %.3f ms" % (e[0].elapsed_time(e[1]) / 20))
k = d.view(torch.int64)
e[0].record()
for _ in range(20):
    torch.sort(k)
e[1].record(); torch.cuda.synchronize()
print("torch.sort 1M int64: %.3f ms" % (e[0].elapsed_time(e[1]) / 20))
e[0].record()
for _ in range(20):
    ep_curve(d, rps)
e[1].record(); torch.cuda.synchronize()
print("ep_curve device timeline per call: %.3f ms" % (e[0].elapsed_time(e[1]) / 20))
# the C entry alone (no Python validation / EPCurve)
import ctypes
from paper_1308_2066_b200 import _native
lib = _native.load()
rp_arr = np.ascontiguousarray(rps, dtype=np.float64)
out = np.empty(rp_arr.size)
st = torch.cuda.current_stream()
for _ in range(5):
    lib.are_pml_many_device(d.data_ptr(), d.numel(), rp_arr.ctypes.data, rp_arr.size, out.ctypes.data, ctypes.c_void_p(st.cuda_stream))
t = []
for _ in range(50):
    t0 = time.perf_counter()
    lib.are_pml_many_device(d.data_ptr(), d.numel(), rp_arr.ctypes.data, rp_arr.size, out.ctypes.data, ctypes.c_void_p(st.cuda_stream))
    t.append(time.perf_counter() - t0)
print("are_pml_many_device alone: median %.3f ms" % (np.median(t) * 1e3))
t = []
for _ in range(50):
    t0 = time.perf_counter()
    torch.sort(d.view(torch.int64)); torch.cuda.synchronize()
    t.append(time.perf_counter() - t0)
print("torch.sort + sync wall: median %.3f ms" % (np.median(t) * 1e3))
