"""GPU: the host-buffer C ABI calls (hire_topk_host / hire_ffn_host — the
calls a reference-side binding makes with plain host pointers). After one
eager call per shape they replay as one captured CUDA graph (H2D copy, the
kernel chain, D2H copy); every call must equal the device-pointer path on
the same inputs, across eager / capture / replay calls, changing inputs,
other ops in between (workspace reuse), and with graphs disabled."""
import ctypes as C

import numpy as np
import pytest
import torch

from tests import _data

pytestmark = pytest.mark.gpu


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _topk_host(H, ctx, z, a, x, cfg):
    B = x.shape[0]
    p = cfg.params()
    cand = np.zeros((B, cfg.k_prime), np.uint32)
    idx = np.zeros((B, cfg.k), np.uint32)
    val = np.zeros((B, cfg.k), np.float32)
    prob = np.zeros((B, cfg.k), np.float32)
    nc, nt, cl = C.c_int64(), C.c_int64(), C.c_int()
    xx = np.ascontiguousarray(x, np.float32)
    H._lib.check(H.lib().hire_topk_host(ctx.h, z.h, a.h, xx.ctypes.data_as(C.c_void_p), B, C.byref(p),
                                        cand.ctypes.data_as(C.c_void_p), idx.ctypes.data_as(C.c_void_p),
                                        val.ctypes.data_as(C.c_void_p), prob.ctypes.data_as(C.c_void_p),
                                        C.byref(nc), C.byref(nt), C.byref(cl)))
    return cand[:, :nc.value], idx[:, :nt.value], val[:, :nt.value], prob[:, :nt.value], bool(cl.value)


@pytest.mark.parametrize("V,d,k,kp,B", [(20000, 256, 16, 256, 2), (6000, 128, 8, 64, 1)])
def test_topk_host_replays_equal_device_path(H, O, V, d, k, kp, B):
    w = _data.lowrank_plus_noise(V, d, 16, V)
    codes, scales = O.quantize_int4(w)
    z = H.ScoreMatrix(T(w))
    a = H.ApproxScorer.quantized(codes, scales)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8)
    ctx = H.Context(0)
    g = np.random.default_rng(1)
    for it in range(6):
        x = (g.standard_normal((B, d)) / np.sqrt(d)).astype(np.float32)
        if it == 3:  # another op on the same context in between (workspace reuse)
            H.topk_select(T(g.standard_normal((3, 50000)).astype(np.float32)), 100, ctx=ctx)
        cand, idx, val, prob, cl = _topk_host(H, ctx, z, a, x, cfg)
        r = H.hire_topk(T(x), z, a, cfg)
        _, pr = H.softmax_topk(z, T(x), a, cfg)
        assert np.array_equal(cand, r.cand.cpu().numpy().astype(np.uint32)), it
        assert np.array_equal(idx, r.top_idx.cpu().numpy().astype(np.uint32)), it
        assert np.array_equal(val.view(np.uint32), r.top_val.cpu().numpy().view(np.uint32)), it
        np.testing.assert_allclose(prob, pr.cpu().numpy(), rtol=1e-6)
        assert cl == r.clamped


def test_ffn_host_replays_equal_device_path(H, O, monkeypatch):
    m, d, k, kp, B = 2048, 256, 102, 204, 3
    u, v = _data.ffn_family(m, d, 5, r=16)
    f = H.GroupedFFN(H.ScoreMatrix(T(u)), H.ScoreMatrix(T(v)))
    a = H.ApproxScorer.quantize(f.u)
    g = np.random.default_rng(2)
    for graphs in ("1", "0"):
        monkeypatch.setenv("HIRE_HOST_GRAPHS", graphs)
        ctx = H.Context(0)
        p = H._lib.FfnParams(k, kp, 1, 1, H.X_INT8, 0, 0)
        for it in range(5):
            x = g.standard_normal((B, d)).astype(np.float32)
            sel = np.zeros((B, k), np.uint32)
            out = np.zeros((B, d), np.float32)
            H._lib.check(H.lib().hire_ffn_host(ctx.h, f.u.h, f.v.h, a.h, x.ctypes.data_as(C.c_void_p), B, C.byref(p),
                                               sel.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
            want, wsel = H.ffn_group_sparse(f, T(x), a, k, kp, x_mode=H.X_INT8)
            assert np.array_equal(sel, wsel.cpu().numpy().astype(np.uint32)), (graphs, it)
            assert np.array_equal(out.view(np.uint32), want.cpu().numpy().view(np.uint32)), (graphs, it)


def test_host_calls_read_pinned_inputs_in_place(H, O):
    """Pinned caller input buffers are read in place: the captured graph's
    fetch kernel takes the address from the context's slot. Alternating pinned buffers, a pageable
    one in between, and a recycled handle address must all give the
    device-path results (no stale pointer in a replayed graph)."""
    V, d, k, kp, B = 20000, 256, 16, 256, 3
    w = _data.lowrank_plus_noise(V, d, 16, 7)
    codes, scales = O.quantize_int4(w)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8)
    ctx = H.Context(0)
    g = np.random.default_rng(3)
    pins = [torch.empty(B, d, dtype=torch.float32).pin_memory().numpy() for _ in range(2)]
    for rnd in range(2):  # a second round with fresh handles (addresses may be reused)
        z = H.ScoreMatrix(T(w))
        a = H.ApproxScorer.quantized(codes, scales)
        for it in range(7):
            x = pins[it % 2] if it != 4 else np.empty((B, d), np.float32)  # it 4: pageable
            x[:] = (g.standard_normal((B, d)) / np.sqrt(d)).astype(np.float32)
            cand, idx, val, prob, cl = _topk_host(H, ctx, z, a, x, cfg)
            r = H.hire_topk(T(x), z, a, cfg)
            assert np.array_equal(idx, r.top_idx.cpu().numpy().astype(np.uint32)), (rnd, it)
            assert np.array_equal(val.view(np.uint32), r.top_val.cpu().numpy().view(np.uint32)), (rnd, it)
        del z, a
    m, kf, kpf = 2048, 102, 204
    u, v = _data.ffn_family(m, d, 9, r=16)
    f = H.GroupedFFN(H.ScoreMatrix(T(u)), H.ScoreMatrix(T(v)))
    fa = H.ApproxScorer.quantize(f.u)
    p = H._lib.FfnParams(kf, kpf, 1, 1, H.X_INT8, 0, 0)
    for it in range(6):
        x = pins[it % 2] if it != 3 else np.empty((B, d), np.float32)
        x[:] = g.standard_normal((B, d)).astype(np.float32)
        sel = np.zeros((B, kf), np.uint32)
        out = np.zeros((B, d), np.float32)
        H._lib.check(H.lib().hire_ffn_host(ctx.h, f.u.h, f.v.h, fa.h, x.ctypes.data_as(C.c_void_p), B, C.byref(p),
                                           sel.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
        want, wsel = H.ffn_group_sparse(f, T(x), fa, kf, kpf, x_mode=H.X_INT8)
        assert np.array_equal(out.view(np.uint32), want.cpu().numpy().view(np.uint32)), it


def test_host_calls_from_two_threads_two_contexts(H, O):
    """Two host threads, one context each (own stream, workspaces and graphs),
    calling hire_topk_host / hire_ffn_host at the same time on shared matrix
    and scorer handles with alternating pinned inputs — the serving pattern
    bench.py's e2e uses. Every call must equal the device-path result of its
    own input: a thread's first call (no CUDA call made on it before) must see
    its buffer's device address, and one context's replay must not disturb
    the other's (round 2e: this pattern faulted when the fetch node was
    re-pointed with cudaGraphExecKernelNodeSetParams)."""
    import threading
    V, d, k, kp, B, lanes, calls = 20000, 256, 16, 256, 4, 2, 60
    w = _data.lowrank_plus_noise(V, d, 16, 11)
    codes, scales = O.quantize_int4(w)
    z = H.ScoreMatrix(T(w))
    a = H.ApproxScorer.quantized(codes, scales)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8)
    m, kf, kpf = 2048, 102, 204
    u, v = _data.ffn_family(m, d, 12, r=16)
    f = H.GroupedFFN(H.ScoreMatrix(T(u)), H.ScoreMatrix(T(v)))
    fa = H.ApproxScorer.quantize(f.u)
    fp = H._lib.FfnParams(kf, kpf, 1, 1, H.X_INT8, 0, 0)
    g = np.random.default_rng(5)

    def pin(shape, dt=torch.float32):
        return torch.empty(shape, dtype=dt).pin_memory().numpy()
    xs, want = [], []
    for i in range(5):
        x = pin((B, d))
        x[:] = (g.standard_normal((B, d)) / np.sqrt(d)).astype(np.float32)
        xs.append(x)
        r = H.hire_topk(T(x), z, a, cfg)
        fo, fs = H.ffn_group_sparse(f, T(x), fa, kf, kpf, x_mode=H.X_INT8)
        want.append((r.top_idx.cpu().numpy().astype(np.uint32), r.top_val.cpu().numpy(), fo.cpu().numpy()))
    torch.cuda.synchronize()
    ctxs = [H.Context(0, torch.cuda.Stream()) for _ in range(lanes)]
    for c in ctxs:  # eager + capture per context, one at a time
        for i in range(3):
            _topk_host(H, c, z, a, xs[i], cfg)
            so, oo = pin((B, kf), torch.int32), pin((B, d))
            H._lib.check(H.lib().hire_ffn_host(c.h, f.u.h, f.v.h, fa.h, xs[i].ctypes.data_as(C.c_void_p), B,
                                               C.byref(fp), so.ctypes.data_as(C.c_void_p),
                                               oo.ctypes.data_as(C.c_void_p)))
    bad = []

    def lane(l):
        ctx = ctxs[l]
        idx, val, prob = pin((B, k), torch.int32).view(np.uint32), pin((B, k)), pin((B, k))
        sel, out = pin((B, kf), torch.int32).view(np.uint32), pin((B, d))
        p = cfg.params()
        n = (C.c_int64(), C.c_int64(), C.c_int())
        ptr = lambda arr: arr.ctypes.data_as(C.c_void_p)  # noqa: E731
        try:
            for i in range(calls):
                j = (i + 2 * l) % len(xs)
                H._lib.check(H.lib().hire_topk_host(ctx.h, z.h, a.h, ptr(xs[j]), B, C.byref(p), None, ptr(idx),
                                                    ptr(val), ptr(prob), *[C.byref(t) for t in n]))
                if not (np.array_equal(idx, want[j][0]) and np.array_equal(val.view(np.uint32), want[j][1].view(np.uint32))):
                    bad.append(("topk", l, i))
                H._lib.check(H.lib().hire_ffn_host(ctx.h, f.u.h, f.v.h, fa.h, ptr(xs[j]), B, C.byref(fp), ptr(sel),
                                                   ptr(out)))
                if not np.array_equal(out.view(np.uint32), want[j][2].view(np.uint32)):
                    bad.append(("ffn", l, i))
        except Exception as e:  # surfaces in the assert below
            bad.append(("error", l, repr(e)))
    th = [threading.Thread(target=lane, args=(l,)) for l in range(lanes)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert not bad, bad[:5]
