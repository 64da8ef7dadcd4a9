"""CPU, world_size 2 over gloo: the DA-TOP-k exchange and merge.

Each rank plays one GPU: it owns the rows [first, first+width) of the width
rule (distributed.hpp:53-57), runs its local stage (here with the oracle on
its shard — the CUDA local stage is checked on the GPU in test_gpu_parity),
encodes its (score, global index) pairs as the same 8-byte rank keys the
device all-gathers, exchanges them with torch.distributed.all_gather, and
merges with the device merge rule. The FFN variant all-reduces partial
down-projections. Results must equal the oracle's single-process da_topk /
da_group_sparse (distributed.hpp:73-206).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inst():
    g = np.random.default_rng(31)
    V, d = 97, 16
    w = g.standard_normal((V, d)).astype(np.float32)
    x = g.standard_normal(d).astype(np.float32)
    u = g.standard_normal((64, d)).astype(np.float32)
    v = g.standard_normal((64, d)).astype(np.float32)
    return w, x, u, v


def _worker(rank, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle as O
    from paper_2402_09360_b200 import parallel as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        w, x, u, v = _inst()
        codes, scales = O.quantize_int4(w)
        scores = O.q4_scores_int8(codes, scales, x, 0)
        results = {}
        for (k, kp, merge, uneven) in [(8, 16, 0, False), (7, 15, 0, True), (8, 16, 1, False),
                                       (5, 9, 1, True)]:
            P.check_divisible(k, kp, WORLD, uneven)
            first, width = P.shard_range(w.shape[0], WORLD, rank)
            kl, kpl = P.quota(k, WORLD, rank), P.quota(kp, WORLD, rank)
            # local stage on this rank's shard (da_topk per-shard step)
            cidx, _, _ = O.topk_select(scores[first:first + width], kpl)
            cidx = np.sort(cidx)
            vals = np.array([O.column_score(w[first + j], x, 0) for j in cidx], dtype=np.float32)
            keys = P.encode_keys(vals, cidx.astype(np.uint64) + first)
            if merge == 0:
                order = np.argsort(keys)[::-1][:kl]
                keys = keys[order]
            slot = (-(-k // WORLD)) if merge == 0 else (-(-kp // WORLD))
            send = np.zeros(slot, dtype=np.uint64)
            send[:keys.size] = keys
            buf = [torch.zeros(slot, dtype=torch.int64) for _ in range(WORLD)]
            dist.all_gather(buf, torch.from_numpy(send.view(np.int64)))
            gathered = np.stack([b.numpy().view(np.uint64) for b in buf])
            K = sum(min(P.quota(k, WORLD, r), P.quota(kp, WORLD, r)) for r in range(WORLD)) if merge == 0 else k
            mv, mi = P.merge_gathered(gathered, K)
            results[(k, kp, merge, uneven)] = (mi.tolist(), mv.tolist())
        # FFN: local select + partial down-projection, all-reduce (sum)
        uc, us = O.quantize_int4(u)
        us_scores = O.q4_scores_int8(uc, us, x, 1)
        fg, wg = P.shard_range(64, WORLD, rank)
        k, kp = 8, 16
        ids, _ = O.ffn_group_sparse(u[fg:fg + wg], v[fg:fg + wg], x, us_scores[fg:fg + wg],
                                    P.quota(k, WORLD, rank), P.quota(kp, WORLD, rank), 1, 1)
        part = O.ffn_apply_groups(u[fg:fg + wg], v[fg:fg + wg], x, ids, 1, 1)
        t = torch.from_numpy(part.copy())
        dist.all_reduce(t)
        allids = [None] * WORLD
        dist.all_gather_object(allids, (ids + fg).tolist())
        results["ffn"] = (sorted(sum(allids, [])), t.numpy().tolist())
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def gloo_results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_da_topk_gloo_matches_oracle(O, gloo_results):
    w, x, u, v = _inst()
    codes, scales = O.quantize_int4(w)
    scores = O.q4_scores_int8(codes, scales, x, 0)
    for (k, kp, merge, uneven) in [(8, 16, 0, False), (7, 15, 0, True), (8, 16, 1, False),
                                   (5, 9, 1, True)]:
        wi, wv, _, _ = O.da_topk(w, x, scores, WORLD, k, kp, 0, merge=merge, uneven=uneven)
        for r in range(WORLD):  # every rank holds the same merged result
            gi, gv = gloo_results[r][(k, kp, merge, uneven)]
            assert gi == wi.tolist() and np.array_equal(np.array(gv, np.float32), wv)


def test_da_group_sparse_gloo_matches_oracle(O, gloo_results):
    w, x, u, v = _inst()
    uc, us = O.quantize_int4(u)
    s = O.q4_scores_int8(uc, us, x, 1)
    ids, out = O.da_group_sparse(u, v, x, s, 8, 16, WORLD)
    for r in range(WORLD):
        gids, gout = gloo_results[r]["ffn"]
        assert gids == ids.tolist()
        # all-reduce sums per-shard partials: same terms, different order
        np.testing.assert_allclose(np.array(gout, np.float32), out, rtol=1e-5, atol=1e-5)


def test_key_encoding_is_the_reference_order():
    from paper_2402_09360_b200 import parallel as P
    g = np.random.default_rng(1)
    vals = g.integers(-3, 4, size=200).astype(np.float32)
    vals[::17] = -0.0
    idx = np.arange(200, dtype=np.uint64)
    keys = P.encode_keys(vals, idx)
    order = np.argsort(keys)[::-1]
    want = sorted(range(200), key=lambda i: (-float(vals[i]), i))  # ranks_before
    assert order.tolist() == want
    dv, di = P.decode_keys(keys)
    assert np.array_equal(di, idx.astype(np.uint32))
    assert np.array_equal(dv, np.where(vals == 0, 0.0, vals).astype(np.float32))


def test_host_rules_match_oracle(O):
    from paper_2402_09360_b200 import parallel as P
    for l in (10, 97, 256000):
        for s in (1, 2, 3, 8):
            for i in range(s):
                assert P.shard_range(l, s, i) == O.partition(l, s, i)
    for k in (410, 820, 128, 7):
        for s in (1, 2, 4, 8):
            assert [P.quota(k, s, i) for i in range(s)] == [O.quota(k, s, i) for i in range(s)]
            assert sum(P.quota(k, s, i) for i in range(s)) == k
