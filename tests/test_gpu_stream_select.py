"""GPU: the stream selector (select2.cuh sel_stream_kernel + sel_fin_kernel:
sample bound and list scan in one launch) against the oracle's topk_select
(linalg.hpp:157-176) and against the pivot + list kernels it replaces.
HIRE_SEL_STREAM=0 disables the path (pivot + list kernels instead); the
default takes it whenever the planner accepts the shape. Bit-exact indices and values, ties by ascending index, on
adversarial rows (the sampler's chunk sees none of the large keys, all keys
equal, ReLU plateaus), ragged lengths (not a multiple of 4 / 128), many
queries, CUDA-graph replay (zero-at-rest counters and tickets)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def N(t):
    return t.cpu().numpy()


def _rows(n, seed):
    g = np.random.default_rng(seed)
    i = np.arange(n)
    rows = {
        "normal": g.standard_normal(n),
        "int_ties": g.integers(-20, 20, size=n),
        "all_equal": np.zeros(n),
        "relu": np.maximum(g.standard_normal(n) - 2.0, 0.0),
        "ascending": np.sort(g.standard_normal(n)),
        "descending": -np.sort(g.standard_normal(n)),
        "spiky": np.where(g.random(n) < 0.001, 100.0 + g.random(n), g.random(n) * 1e-3),
        # every large key sits in granules the first chunks never own
        "one_chunk": np.where((i // 128) % 16 == 7, 10.0 + g.random(n), g.random(n)),
        "head_heavy": np.where(i < n // 50, 5.0 + g.random(n), g.random(n)),
        "neg": -np.abs(g.standard_normal(n)) - 1.0,
    }
    return {k: v.astype(np.float32) for k, v in rows.items()}


def _check(H, O, v, k):
    idx, val, cl = H.topk_select(T(v), k)
    for b in range(v.shape[0]):
        wi, wv, wcl = O.topk_select(v[b], k)
        assert np.array_equal(N(idx[b]).astype(np.uint32), wi), (b, k)
        assert np.array_equal(N(val[b]).view(np.uint32), wv.view(np.uint32))
        assert cl == wcl


@pytest.fixture
def stream(monkeypatch):
    monkeypatch.setenv("HIRE_SEL_STREAM", "1")


@pytest.mark.parametrize("kind", ["normal", "int_ties", "all_equal", "relu", "ascending", "descending", "spiky",
                                  "one_chunk", "head_heavy", "neg"])
@pytest.mark.parametrize("n,k", [(150000, 1000), (262147, 1024), (40001, 300)])
def test_stream_select_matches_oracle(H, O, stream, kind, n, k):
    v = np.stack([_rows(n, 11)[kind], _rows(n, 12)[kind], _rows(n, 13)[kind]])
    _check(H, O, v, k)


@pytest.mark.parametrize("B", [1, 16, 40])
def test_stream_select_batches_and_default_gate(H, O, B):
    # the stream path by default (no env)
    n, k = 70000, 512
    g = np.random.default_rng(3)
    v = g.standard_normal((B, n)).astype(np.float32)
    v[B // 2] = np.round(v[B // 2] * 4) / 4  # one row full of ties
    _check(H, O, v, k)


@pytest.mark.parametrize("n,k,B", [(9000, 128, 1), (32768, 256, 1), (32000, 128, 16), (64000, 1024, 4)])
def test_stream_default_gate_short_rows(H, O, n, k, B):
    # short rows and small batches take the stream path too (no size gate since
    # round 2d); random rows stay off the finisher's slow path
    g = np.random.default_rng(21)
    v = g.standard_normal((B, n)).astype(np.float32)
    ctx = H.default_context()
    before = ctx.select_fallbacks()
    _check(H, O, v, k)
    assert ctx.select_fallbacks() == before


def test_stream_equals_pivot_list_path(H, O, monkeypatch):
    n, k, B = 131072 + 4, 2048, 9
    g = np.random.default_rng(5)
    v = (g.standard_normal((B, n)) * g.random((B, 1)) * 3).astype(np.float32)
    monkeypatch.setenv("HIRE_SEL_STREAM", "1")
    i1, v1, _ = H.topk_select(T(v), k)
    monkeypatch.setenv("HIRE_SEL_STREAM", "0")
    i0, v0, _ = H.topk_select(T(v), k)
    assert torch.equal(i1, i0) and torch.equal(v1, v0)


def test_stream_select_graph_replay(H, O, stream):
    # counters, bounds and tickets are zero at rest: a captured call replays
    # on new data without re-initialisation, and after a fallback
    n, k, B = 100000, 700, 4
    ctx = H.default_context()
    buf = torch.zeros(B, n, device="cuda")
    s = torch.cuda.Stream()
    g = np.random.default_rng(8)
    rows = [g.standard_normal((B, n)).astype(np.float32),
            np.zeros((B, n), np.float32),  # all equal: every key listed -> overflow -> exact fallback
            g.standard_normal((B, n)).astype(np.float32)]
    with torch.cuda.stream(s):
        buf.copy_(T(rows[0]))
        H.topk_select(buf, k)
        s.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            idx, val, _ = H.topk_select(buf, k)
        for r in rows:
            buf.copy_(T(r))
            gr.replay()
            s.synchronize()
            for b in range(B):
                wi, wv, _ = O.topk_select(r[b], k)
                assert np.array_equal(N(idx[b]).astype(np.uint32), wi)
                assert np.array_equal(N(val[b]).view(np.uint32), wv.view(np.uint32))
    del ctx


def test_stream_no_fallback_on_benign_rows(H, stream):
    # the bound holds on exchangeable rows: the finisher never takes its slow
    # path (device trace of query 0)
    n, k, B = 256000, 1024, 8
    g = torch.Generator(device="cuda").manual_seed(4)
    ctx = H.default_context()
    for _ in range(5):
        v = torch.randn(B, n, device="cuda", generator=g)
        H.topk_select(v, k)
        torch.cuda.synchronize()
        ctx.ktrace(1)
        H.topk_select(v, k)
        torch.cuda.synchronize()
        sp = ctx.ktrace(2)
        ctx.ktrace(0)
        assert sp.get("fin_fallback", 0) == 0
        assert k <= sp.get("fin_listed", 0) <= 8192
        assert "pivot" not in sp  # one launch for bound + scan


def test_fallback_counter_and_bound_rate(H, stream):
    # hire_ctx_select_fallbacks: the slow whole-row path is counted per query.
    # A constant row overflows every list segment (one fallback per query);
    # exchangeable rows (normal, heavy-tailed, bimodal) never miss the bound:
    # 60 batches x 32 queries without a single fallback (designed rate 1e-7 per query)
    ctx = H.default_context()
    n, k, B = 256000, 1024, 32
    f0 = ctx.select_fallbacks()
    H.topk_select(torch.zeros(3, 150000, device="cuda"), 500)
    assert ctx.select_fallbacks() - f0 == 3
    g = torch.Generator(device="cuda").manual_seed(7)
    f1 = ctx.select_fallbacks()
    for it in range(60):
        v = torch.randn(B, n, device="cuda", generator=g)
        if it % 3 == 1:
            v = torch.exp(1.5 * v)  # log-normal
        elif it % 3 == 2:
            v = v + 3.0 * (torch.rand(B, n, device="cuda", generator=g) < 0.01)  # 1 % of the rows shifted up
        H.topk_select(v, k)
    assert ctx.select_fallbacks() - f1 == 0
