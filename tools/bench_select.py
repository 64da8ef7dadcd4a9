"""Times hire_topk_select (exact top-k of B score rows of n keys) with the
stream selector forced on / off, CUDA events over a captured graph of 20
calls. Decides the row-length / batch rule of run_select (hire_cuda.cu)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_09360_b200 as H  # noqa: E402


def timed(scores, k, ctx, s):
    with torch.cuda.stream(s):
        H.topk_select(scores, k, ctx=ctx)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        n = 20
        with torch.cuda.graph(graph, stream=s):
            for _ in range(n):
                H.topk_select(scores, k, ctx=ctx)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    s = torch.cuda.Stream()
    ctx = H.Context(0, s)
    for n in (9000, 12000, 16384, 32000, 32768, 64000, 128000):
        for B in (1, 4, 16, 32):
            for k in (128, 256, 1024):
                if n * B >= 1 << 20:
                    continue
                scores = torch.randn(B, n, device="cuda", generator=g)
                r = {"n": n, "B": B, "k": k}
                for mode in ("0", "1"):
                    os.environ["HIRE_SEL_STREAM"] = mode
                    r["stream" if mode == "1" else "list"] = round(timed(scores, k, ctx, s), 2)
                fb = ctx.select_fallbacks()
                r["fallbacks"] = fb
                print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
