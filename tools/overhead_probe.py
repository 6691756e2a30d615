import os, sys, time, statistics
sys.path.insert(0, "/root/repo")
from paper_2405_13364_b200 import veil
import ctypes as C
from paper_2405_13364_b200.abi import default_params
sc = veil.Scene.workload("stack64k", 2)
L = veil.lib()
p = default_params()
for _ in range(10): veil.render_device(sc)
N = 200
t = time.perf_counter()
for _ in range(N): L.veil_render_device(sc.h, C.byref(p), None)
wall = (time.perf_counter() - t) / N * 1e3
dev = statistics.median(veil.render_device(sc).total_ms for _ in range(20))
print(f"stack64k wall/call {wall:.4f} ms, device {dev:.4f} ms, host overhead {wall-dev:.4f} ms")
sc2 = veil.Scene.synthetic("layered_quads", 1, 64, 64)
for _ in range(10): veil.render_device(sc2)
t = time.perf_counter()
for _ in range(N): L.veil_render_device(sc2.h, C.byref(p), None)
wall = (time.perf_counter() - t) / N * 1e3
dev = statistics.median(veil.render_device(sc2).total_ms for _ in range(20))
print(f"tiny scene wall/call {wall:.4f} ms, device {dev:.4f} ms, overhead {wall-dev:.4f} ms")
