"""Device timeline of one step of a bench workload (debug aid, not a bench
number): replays the step in a CUDA graph a few times, then once more with
the %globaltimer kernel trace on (hire_debug_ktrace), and prints each
kernel's [first CTA start, last CTA end] in microseconds.

  python tools/ktrace.py --workload cfg3 --batch 1 [--reps 3]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--select", default="exact")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import paper_2402_09360_b200 as H
    H.lib()
    wl = bench.make_workload(args)
    wl.attach(H)
    xs = wl.inputs(8)
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        ctx = H.default_context()
        for i in range(4):
            wl.step(i, xs[i])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            wl.step(5, xs[5])
    for r in range(args.reps):
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ctx.ktrace(1)
        g.replay()
        torch.cuda.synchronize()
        spans = ctx.ktrace(2)
        ctx.ktrace(0)
        end = max(v[1] for v in spans.values() if isinstance(v, tuple))
        print(json.dumps({"workload": args.workload, "batch": args.batch, "rep": r, "step_span_us": end,
                          "spans": spans}))


if __name__ == "__main__":
    main()
