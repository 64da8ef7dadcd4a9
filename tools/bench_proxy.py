"""Times the int4 proxy kernel alone (hire_scores, int8 x) at cfg3's shape
(V=256000, d=2048) for several batch sizes, with CUDA events over a
captured graph of N launches; 4 proxies cycled so every launch streams
from HBM. HIRE_UMMA_MIN_B selects the kernel family (0 = mma.sync path).
Prints one JSON line per batch size."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_09360_b200 as H  # noqa: E402


def main():
    V, d = int(os.environ.get("V", 256000)), int(os.environ.get("D", 2048))
    batches = [int(b) for b in os.environ.get("BATCHES", "16,32,64").split(",")]
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    g = torch.Generator(device="cuda").manual_seed(0)
    scorers = []
    for _ in range(4):
        W = (torch.randn(V, d, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
        scorers.append(H.ApproxScorer.quantize(H.ScoreMatrix(W)))
        del W
    torch.cuda.synchronize()
    for B in batches:
        x = torch.randn(B, d, device="cuda", generator=g)
        outs = [torch.empty(B, V, device="cuda") for _ in range(4)]
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ctx = H.Context(0, s)
            for a in scorers:
                a.scores(x, x_mode=H.X_INT8, ctx=ctx)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            n = 40
            with torch.cuda.graph(graph, stream=s):
                for i in range(n):
                    scorers[i % 4].scores(x, x_mode=H.X_INT8, ctx=ctx)
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / n
        bytes_ = V * (d // 2 + 4)
        print(json.dumps({"B": B, "V": V, "d": d, "umma_min_b": os.environ.get("HIRE_UMMA_MIN_B", "default"),
                          "us_per_launch": round(us, 2), "gbs": round(bytes_ / us / 1e3, 1),
                          "frac": round(bytes_ / us / 1e3 / peak, 4)}), flush=True)


if __name__ == "__main__":
    main()
