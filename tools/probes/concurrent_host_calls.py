"""Two host threads, one hire context each, calling hire_topk_host concurrently
on shared matrix / scorer handles (debug probe for cross-context races).

  python tools/probes/concurrent_host_calls.py [V d B kp k calls lanes]
"""
import ctypes as C
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2402_09360_b200 as H  # noqa: E402


def main():
    a = [int(v) for v in sys.argv[1:]]
    V, d, B, kp, k, calls, lanes = (a + [32000, 512, 8, 256, 32, 200, 2][len(a):])[:7]
    H.lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    Wt = (torch.randn(V, 32, generator=g, device="cuda") @ torch.randn(32, d, generator=g, device="cuda") / 32 ** 0.5
          + 0.1 * torch.randn(V, d, generator=g, device="cuda")).to(torch.bfloat16)
    W = H.ScoreMatrix(Wt)
    A = H.ApproxScorer.quantize(W)
    mode = os.environ.get("PROBE_MODE", "")
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_FP32 if mode == "fp32" else H.X_INT8)

    def pinned(shape, dt):
        return torch.empty(shape, dtype=dt).pin_memory().numpy()
    xs = []
    for i in range(8):
        x = pinned((B, d), torch.float32)
        x[:] = torch.randn(B, d, generator=g, device="cuda").cpu().numpy()
        xs.append(x)
    addr = lambda arr: C.c_void_p(arr.ctypes.data)  # noqa: E731
    lw = []
    if mode == "devgraph":  # hire_topk_run captured in one torch CUDA graph per lane, replayed concurrently
        xd = torch.from_numpy(xs[0]).cuda()
        gl = []
        for l in range(lanes):
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                ctx = H.Context(0, st)
                for _ in range(3):
                    r = H.softmax_topk(W, xd, A, cfg, ctx=ctx)
                torch.cuda.synchronize()
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=st):
                    r = H.softmax_topk(W, xd, A, cfg, ctx=ctx)
            gl.append((gr, r, ctx, st))
        torch.cuda.synchronize()

        def dlane(l):
            for _ in range(calls):
                gl[l][0].replay()
                gl[l][3].synchronize()
        th = [threading.Thread(target=dlane, args=(l,)) for l in range(lanes)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()
        print("devgraph ok; mismatching calls per lane: n/a")
        return
    Ws, As = [W], [A]
    if mode == "ownhandles":
        for l in range(1, lanes):
            Ws.append(H.ScoreMatrix(Wt.clone()))
            As.append(H.ApproxScorer.quantize(Ws[-1]))
    for l in range(lanes):
        lw.append(dict(W=Ws[l % len(Ws)], A=As[l % len(As)], ctx=H.Context(0, torch.cuda.Stream()), idx=pinned((B, k), torch.int32),
                       val=pinned((B, k), torch.float32), prob=pinned((B, k), torch.float32),
                       p=cfg.params(), n=(C.c_int64(), C.c_int64(), C.c_int())))

    fixed = os.environ.get("PROBE_FIXED_X") == "1"  # every lane keeps one input buffer (no fetch-node re-pointing)

    def call(l, i):
        s = lw[l]
        if fixed:
            i = l
        H._lib.check(H.lib().hire_topk_host(s["ctx"].h, s["W"].h, s["A"].h, addr(xs[i % 8]), B, C.byref(s["p"]), None,
                                            addr(s["idx"]), addr(s["val"]), None if mode == "noprob" else addr(s["prob"]),
                                            *[C.byref(v) for v in s["n"]]))
        return s["idx"].copy(), s["val"].copy()

    want = [call(0, i) for i in range(8)]
    for l in range(lanes):
        for i in range(8):
            call(l, i)
    bad = [0] * lanes
    if mode == "mainsleep":  # main thread only, idle gaps between calls
        import time
        nb = 0
        for i in range(40):
            time.sleep(0.005 if i % 2 else 0.0)
            gi, gv = call(0, i)
            if not np.array_equal(gi, want[i % 8][0]):
                nb += 1
                print("main call", i, "mismatch; equals", [j for j in range(8) if np.array_equal(gi, want[j][0])])
        print("mainsleep mismatches:", nb)
        return

    def lane(l):
        for i in range(calls):
            gi, gv = call(l, i)
            if fixed:
                i = l
            if not (np.array_equal(gi, want[i % 8][0]) and np.array_equal(gv.view(np.uint32), want[i % 8][1].view(np.uint32))):
                bad[l] += 1
                which = [j for j in range(8) if np.array_equal(gi, want[j][0])]
                print(f"lane {l} call {i}: idx equal {np.array_equal(gi, want[i % 8][0])}; equals want of input {which}", flush=True)
    th = [threading.Thread(target=lane, args=(l,)) for l in range(lanes)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    print("mismatching calls per lane:", bad)


if __name__ == "__main__":
    main()
