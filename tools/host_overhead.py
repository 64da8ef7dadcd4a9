"""Where the time of a host-buffer call goes (debug aid): per-call wall time
of hire_topk_host against the device-only step, an empty graph launch + sync,
and a pinned H2D + D2H pair + sync, at cfg3's shapes."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2402_09360_b200 as H  # noqa: E402


def wall(fn, n=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


class A:
    workload, batch, select = "cfg3", int(os.environ.get("B", "1")), "exact"


def pin(shape, dt):
    return torch.empty(shape, dtype=dt).pin_memory().numpy()


wl = bench.make_workload(A)
wl.attach(H)
wl.host_buffers(pin)
xh = pin((wl.B, wl.d), torch.float32)
xh[:] = wl.inputs(1)[0].cpu().numpy()
oa = pin((wl.B, wl.k), torch.int32).view(np.uint32)
ob = pin((wl.B, wl.k), torch.float32)
res = {}
for own in (0, 1):
    ctx = H.Context(0) if not own else None
    if own:
        h = C.c_void_p()
        H._lib.check(H.lib().hire_ctx_create(0, None, 1, C.byref(h)))
        ctx = type("Ctx", (), {"h": h})()
    res[f"topk_host_us(own_stream={own})"] = wall(lambda: wl.host_step(0, xh, oa, ob, ctx))
xd = torch.from_numpy(xh).cuda()
res["device_call_us(eager launches)"] = wall(lambda: wl.step(0, xd))
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
a = torch.zeros(1, device="cuda")
with torch.cuda.graph(g, stream=s):
    a.add_(1)
res["tiny_graph_launch_sync_us"] = wall(lambda: (g.replay(), torch.cuda.current_stream().synchronize()))
hp = torch.empty(wl.B * wl.d, dtype=torch.float32).pin_memory()
dp = torch.empty_like(hp, device="cuda")
ho = torch.empty(wl.B * 128, dtype=torch.float32).pin_memory()
do = torch.empty_like(ho, device="cuda")


def copies():
    dp.copy_(hp, non_blocking=True)
    ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().synchronize()


res["h2d_x_d2h_result_sync_us"] = wall(copies)
print(res)
