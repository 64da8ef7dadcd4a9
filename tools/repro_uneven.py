"""Repro helper: DA-TOP-k with uneven quotas (tests/test_gpu_parity.py::
test_da_topk_uneven_quotas) in a fresh process; prints mismatches."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tests import _data  # noqa: E402
import oracle as O  # noqa: E402
import paper_2402_09360_b200 as H  # noqa: E402

O.build()
V, d, k, kp, s = 9000, 1024, 410, 820, 8
w = _data.lowrank_plus_noise(V, d, 32, 61)
codes, scales = O.quantize_int4(w)
z = H.ScoreMatrix(torch.from_numpy(w).cuda())
a = H.ApproxScorer.quantized(codes, scales)
x = _data.queries(1, d, 19)
cfg = H.HireConfig(k=k, k_prime=kp, x_mode=H.X_INT8, strict=True)
for rep in range(3):
    ti, tv, _ = H.da_topk_emulated(z, a, torch.from_numpy(x).cuda(), s, cfg, uneven=True)
    scores = O.q4_scores_int8(codes, scales, x[0], 0)
    wi, wv, _, _ = O.da_topk(w, x[0], scores, s, k, kp, 0, uneven=True)
    gi = ti[0].cpu().numpy().astype(np.uint32)
    bad = np.nonzero(gi != wi)[0]
    print("rep", rep, "mismatches", len(bad), "pos", bad[:10].tolist(), "got", gi[bad[:5]].tolist(),
          "want", wi[bad[:5]].tolist(), "got_in_want", [int(v in set(wi.tolist())) for v in gi[bad[:5]]])
