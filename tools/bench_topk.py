"""Times hire_topk (cfg3 shape: V=256000, d=2048, int4 proxy x int8 x,
k'=1024, k=64) for several batch sizes with CUDA events over a captured
graph; 4 vocab copies cycled so every call streams from HBM. Env: BATCHES,
HIRE_FSEL (u = tcgen05 proxy without the fused pre-selection)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_09360_b200 as H  # noqa: E402


def main():
    V, d = int(os.environ.get("V", 256000)), int(os.environ.get("D", 2048))
    batches = [int(b) for b in os.environ.get("BATCHES", "16,32").split(",")]
    g = torch.Generator(device="cuda").manual_seed(0)
    mats = []
    for _ in range(int(os.environ.get("COPIES", 4))):
        W = (torch.randn(V, d, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
        z = H.ScoreMatrix(W)
        mats.append((z, H.ApproxScorer.quantize(z)))
    cfg = H.HireConfig(k=64, k_prime=1024, x_mode=H.X_INT8)
    torch.cuda.synchronize()
    for B in batches:
        x = torch.randn(B, d, device="cuda", generator=g) / d ** 0.5
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ctx = H.Context(0, s)
            for z, a in mats:
                H.hire_topk(x, z, a, cfg, ctx=ctx, want_candidates=False)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            n = 20
            with torch.cuda.graph(graph, stream=s):
                for i in range(n):
                    z, a = mats[i % len(mats)]
                    H.hire_topk(x, z, a, cfg, ctx=ctx, want_candidates=False)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"B": B, "fsel": os.environ.get("HIRE_FSEL", "default"),
                          "us_per_call": round(e0.elapsed_time(e1) * 1e3 / n, 2)}), flush=True)


if __name__ == "__main__":
    main()
