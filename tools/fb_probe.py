"""Debug aid: how often, and on which inputs, a bench workload takes the
selector's slow exact path (hire_ctx_select_fallbacks deltas per step).
  python tools/fb_probe.py cfg4 16 [steps]"""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2402_09360_b200 as H
H.lib()
class A: workload, batch, select = sys.argv[1], int(sys.argv[2]), "exact"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5000
wl = bench.make_workload(A); wl.attach(H)
ctx = H.default_context()
xs = wl.inputs(50)
f0 = ctx.select_fallbacks()
hits = collections.Counter()
for i in range(steps):
    wl.step(i, xs[i % 50])
    f = ctx.select_fallbacks()
    if f != f0:
        hits[i % 50] += f - f0; f0 = f
print("steps", steps, "fallbacks by input:", dict(hits))
import ctypes as C
for j in list(hits)[:2]:
    f0 = ctx.select_fallbacks()
    for _ in range(200): wl.step(0, xs[j])
    print("input", j, "repeated 200x:", ctx.select_fallbacks() - f0)
    for _ in range(400):
        f0 = ctx.select_fallbacks()
        ctx.ktrace(1); wl.step(0, xs[j]); torch.cuda.synchronize()
        buf = (C.c_ulonglong * 96)()
        H._lib.check(H.lib().hire_debug_ktrace(ctx.h, 2, buf, 96))
        ctx.ktrace(0)
        if ctx.select_fallbacks() != f0:
            print("fallback: total_raw=%x tau=%x T=%x reason=%d b=%d" % (buf[84], buf[85], buf[86], buf[87], buf[88]))
            break
