"""Where the time of a cfg2 host-buffer call (hire_ffn_host) goes (debug
aid): per-call wall time cycling the layers vs one layer, the device-only
graphed step + sync, and the Python/ctypes marshalling alone."""
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


def wall(fn, n=300):
    for _ in range(30):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


class A:
    workload, batch, select = "cfg2", 8, "exact"


def main():
    wl = bench.make_workload(A)
    wl.attach(H)
    ctx = H.Context(0)
    pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory().numpy()
    xh = pin((wl.B, wl.d), torch.float32)
    xh[:] = np.random.default_rng(0).standard_normal((wl.B, wl.d)) / np.sqrt(wl.d)
    sel = pin((wl.B, wl.k), torch.int32).view(np.uint32)
    out = pin((wl.B, wl.d), torch.float32)
    it = [0]

    def cyc():
        wl.host_step(it[0], xh, sel, out, ctx)
        it[0] += 1

    res = {"n_layers": len(wl.layers)}
    res["host_call_cycling_us"] = wall(cyc)
    res["host_call_one_layer_us"] = wall(lambda: wl.host_step(0, xh, sel, out, ctx))
    f, a = wl.layers[0]
    p = H._lib.FfnParams(wl.k, wl.kp, 1, 1, H.X_INT8, 0, 0)
    xp, sp, op = (xh.ctypes.data_as(C.c_void_p), sel.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
    res["host_call_prebound_us"] = wall(lambda: H.lib().hire_ffn_host(ctx.h, f.u.h, f.v.h, a.h, xp, wl.B, C.byref(p), sp, op))
    res["marshal_only_us"] = wall(lambda: (H._lib.FfnParams(wl.k, wl.kp, 1, 1, H.X_INT8, 0, 0), xh.ctypes.data_as(C.c_void_p),
                                          sel.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
    xd = torch.from_numpy(xh).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        wl.step(0, xd)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            wl.step(0, xd)

    def rep():
        g.replay()
        torch.cuda.synchronize()
    res["device_graph_replay_sync_us"] = wall(rep)
    print(res)


if __name__ == "__main__":
    main()
