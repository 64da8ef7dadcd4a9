"""The multi-rank DA-TOP-k / DA-FFN path through the C ABI, on one GPU.

* hire_da_topk_run / hire_da_ffn_run with a 1-rank NCCL communicator: the
  full local -> ncclAllGather -> merge chain runs (the bench's N = 1 and the
  driver's single-GPU box can execute every NCCL call site); results equal
  hire_topk / ffn_group_sparse (the reference's s = 1 equivalence,
  test_distributed.cpp:104-117) and the single-GPU emulation.
* Two processes, each one rank (world 2) on the same GPU: each runs
  hire_da_topk_local / hire_da_ffn_local on its own shard (rows of the width
  rule, distributed.hpp:53-57), the device-produced keys / partials travel
  through torch.distributed (gloo) on the host, and hire_*_merge runs on every
  rank. No kernel of one process waits on the other (the exchange is on the
  host), so the two processes need not be co-scheduled. Both ranks' results
  must equal hire_da_topk_emulated / hire_da_ffn_emulated bit for bit, and
  the oracle's da_topk in strict mode.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from tests import _data

pytestmark = pytest.mark.gpu


def T(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype)


def _q4(H, O, V, d, seed):
    w = _data.lowrank_plus_noise(V, d, 16, seed)
    codes, scales = O.quantize_int4(w)
    return w, H.ScoreMatrix(T(w)), H.ApproxScorer.quantized(codes, scales), codes, scales


@pytest.mark.parametrize("merge", [0, 1])
@pytest.mark.parametrize("strict", [False, True])
def test_da_topk_run_nccl_one_rank(H, O, merge, strict):
    from paper_2402_09360_b200 import parallel as P
    V, d, k, kp, B = 20000, 1024, 64, 512, 3
    w, z, a, codes, scales = _q4(H, O, V, d, 71)
    x = _data.queries(B, d, 72)
    cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8, strict=strict)
    comm = P.Communicator(1, 0)
    ti, tv, _ = P.da_topk(z, a, V, T(x), cfg, comm, merge=merge)       # local -> ncclAllGather -> merge
    ei, ev, _ = H.da_topk_emulated(z, a, T(x), 1, cfg, merge=merge)
    r = H.hire_topk(T(x), z, a, cfg)
    assert torch.equal(ti, ei) and torch.equal(tv.view(torch.int32), ev.view(torch.int32))
    assert torch.equal(ti, r.top_idx) and torch.equal(tv.view(torch.int32), r.top_val.view(torch.int32))
    if strict:
        for b in range(B):
            wi, wv, _, _ = O.da_topk(w, x[b], O.q4_scores_int8(codes, scales, x[b], 0), 1, k, kp, 0, merge=merge)
            assert np.array_equal(ti[b].cpu().numpy().astype(np.uint32), wi)
            assert np.array_equal(tv[b].cpu().numpy().view(np.uint32), wv.view(np.uint32))


def test_da_ffn_run_nccl_one_rank(H, O):
    from paper_2402_09360_b200 import parallel as P
    m, d, k, kp, B = 2048, 1024, 128, 256, 3
    u, v = _data.ffn_family(m, d, 73, r=32)
    codes, scales = O.quantize_int4(u)
    f = H.GroupedFFN(H.ScoreMatrix(T(u)), H.ScoreMatrix(T(v)), 1, "relu")
    a = H.ApproxScorer.quantized(codes, scales)
    x = _data.queries(B, d, 74, scale=1.0)
    comm = P.Communicator(1, 0)
    out, sel = P.da_group_sparse(f, a, m, T(x), k, kp, comm, x_mode=H.X_INT8)   # all-gather + rank-order sum
    o2, s2 = H.ffn_group_sparse(f, T(x), a, k, kp, x_mode=H.X_INT8)
    assert torch.equal(sel, s2)
    assert torch.equal(out, o2)  # == as floats (0 + -0 = +0)
    o3, s3 = P.da_group_sparse(f, a, m, T(x), k, kp, None, x_mode=H.X_INT8)     # no communicator
    assert torch.equal(s3, s2) and torch.equal(o3, o2)


# ------------------------------------------------------------ two ranks ---
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [  # (k, k_prime, merge, uneven, strict)
    (64, 512, 0, False, True), (64, 512, 1, False, True), (63, 511, 0, True, True), (64, 512, 1, False, False)]


def _rank_main(rank, world, port, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import oracle as O
    import paper_2402_09360_b200 as H
    from paper_2402_09360_b200 import parallel as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        V, d, B = 30001, 1024, 12  # B >= 9: the local proxy runs on the tcgen05 kernel
        w = _data.lowrank_plus_noise(V, d, 16, 75)
        codes, scales = O.quantize_int4(w)
        f0, wd = P.shard_range(V, world, rank)
        z = H.ScoreMatrix(T(w[f0:f0 + wd]))
        a = H.ApproxScorer.quantized(codes[f0:f0 + wd], scales[f0:f0 + wd])
        x = T(_data.queries(B, d, 76))
        res = {}
        for ci, (k, kp, merge, uneven, strict) in enumerate(CASES):
            cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8, strict=strict)
            send = P.da_topk_local(z, a, V, world, rank, x, cfg, merge=merge, uneven=uneven).cpu()
            bufs = [torch.zeros_like(send) for _ in range(world)]
            dist.all_gather(bufs, send)
            g = torch.stack(bufs).cuda()
            ti, tv, _ = P.da_topk_merge(g, V, world, cfg, merge=merge, uneven=uneven)
            res[f"ti{ci}"], res[f"tv{ci}"] = ti.cpu().numpy(), tv.cpu().numpy()
        # FFN over hidden-unit shards
        m, kf, kpf = 4096, 256, 512
        u, v = _data.ffn_family(m, d, 77, r=32)
        uc, us = O.quantize_int4(u)
        fg, wg = P.shard_range(m, world, rank)
        fs = H.GroupedFFN(H.ScoreMatrix(T(u[fg:fg + wg])), H.ScoreMatrix(T(v[fg:fg + wg])), 1, "relu")
        fa = H.ApproxScorer.quantized(uc[fg:fg + wg], us[fg:fg + wg])
        xf = T(_data.queries(B, d, 78, scale=1.0))
        sel, part = P.da_ffn_local(fs, fa, m, world, rank, xf, kf, kpf, x_mode=H.X_INT8)
        sel, part = sel.cpu(), part.cpu()
        sb = [torch.zeros_like(sel) for _ in range(world)]
        pb = [torch.zeros_like(part) for _ in range(world)]
        dist.all_gather(sb, sel)
        dist.all_gather(pb, part)
        out, usel = P.da_ffn_merge(torch.stack(sb).cuda(), torch.stack(pb).cuda(), m, kf, 1)
        res["ffn_out"], res["ffn_sel"] = out.cpu().numpy(), usel.cpu().numpy()
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


def test_da_two_processes_exchange_on_host(H, O):
    import torch.multiprocessing as mp
    world = 2
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_rank_main, args=(world, _free_port(), td), nprocs=world, join=True)
        got = [dict(np.load(os.path.join(td, f"rank{r}.npz"))) for r in range(world)]
    V, d, B = 30001, 1024, 12
    w = _data.lowrank_plus_noise(V, d, 16, 75)
    codes, scales = O.quantize_int4(w)
    z = H.ScoreMatrix(T(w))
    a = H.ApproxScorer.quantized(codes, scales)
    xn = _data.queries(B, d, 76)
    for ci, (k, kp, merge, uneven, strict) in enumerate(CASES):
        cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8, strict=strict)
        ei, ev, _ = H.da_topk_emulated(z, a, T(xn), world, cfg, merge=merge, uneven=uneven)
        for r in range(world):
            assert np.array_equal(got[r][f"ti{ci}"], ei.cpu().numpy()), (ci, r)
            assert np.array_equal(got[r][f"tv{ci}"].view(np.uint32), ev.cpu().numpy().view(np.uint32)), (ci, r)
        if strict:
            for b in range(B):
                wi, wv, _, _ = O.da_topk(w, xn[b], O.q4_scores_int8(codes, scales, xn[b], 0), world, k, kp, 0,
                                         merge=merge, uneven=uneven)
                assert np.array_equal(got[0][f"ti{ci}"][b].astype(np.uint32), wi), (ci, b)
                assert np.array_equal(got[0][f"tv{ci}"][b].view(np.uint32), wv.view(np.uint32)), (ci, b)
    m, kf, kpf = 4096, 256, 512
    u, v = _data.ffn_family(m, d, 77, r=32)
    uc, us = O.quantize_int4(u)
    f = H.GroupedFFN(H.ScoreMatrix(T(u)), H.ScoreMatrix(T(v)), 1, "relu")
    fa = H.ApproxScorer.quantized(uc, us)
    xf = _data.queries(B, d, 78, scale=1.0)
    eo, es = H.da_group_sparse_emulated(f, T(xf), fa, kf, kpf, world, x_mode=H.X_INT8)
    for r in range(world):
        assert np.array_equal(got[r]["ffn_sel"], es.cpu().numpy()), r
        assert np.array_equal(got[r]["ffn_out"].view(np.uint32), eo.cpu().numpy().view(np.uint32)), r
    for b in range(B):  # the reference's union sum order differs: tolerance
        ids, want = O.da_group_sparse(u, v, xf[b], O.q4_scores_int8(uc, us, xf[b], 1), kf, kpf, world)
        assert np.array_equal(got[0]["ffn_sel"][b].astype(np.uint32), ids)
        np.testing.assert_allclose(got[0]["ffn_out"][b], want, rtol=1e-4, atol=1e-4 * np.abs(want).max())


def test_bench_da_flow_one_rank_nccl():
    """bench.py's N > 1 flow (da_topk -> ncclAllGather -> merge captured in a CUDA
    graph, staged profiling, device timeline, e2e with pinned copies) on one
    GPU with a 1-rank communicator (HIRE_BENCH_DA=1): the line must carry
    every contract key and the DA step must not lose more than the merge to
    the single-GPU call."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HIRE_BENCH_DA="1")
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "4", "--warmup", "3",
                        "--no-cpu-baseline"], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "ms_per_step", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert "1-rank NCCL" in line["config"]["parallelism"]
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["e2e"]["path"].startswith("python parallel.da_topk")
