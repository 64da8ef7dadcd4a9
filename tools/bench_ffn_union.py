"""Time one HiRE-FFN layer (cfg2 shape: m=8192, d=2048, bf16, k'=820, k=410,
int8 x) with the batch-union gather on / off, per batch size (CUDA graph of
20 layers over 4 weight copies, CUDA events).

  python tools/bench_ffn_union.py [--batches 8,16,32,64]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="8,16,32,64")
    ap.add_argument("--modes", default="0,1")
    args = ap.parse_args()
    import paper_2402_09360_b200 as H
    H.lib()
    m, d, k, kp = 8192, 2048, 410, 820
    g = torch.Generator(device="cuda").manual_seed(0)
    layers = []
    for _ in range(4):
        def one():
            base = torch.randn(m, d, device="cuda", generator=g) / d ** 0.5
            A = torch.randn(m, 128, device="cuda", generator=g)
            Bm = torch.randn(128, d, device="cuda", generator=g)
            return (base + 3.0 * (A @ Bm) / (128 * d) ** 0.5).to(torch.bfloat16)
        f = H.GroupedFFN(H.ScoreMatrix(one()), H.ScoreMatrix(one()), 1)
        layers.append((f, H.ApproxScorer.quantize(f.u)))
    s = torch.cuda.Stream()
    for B in [int(b) for b in args.batches.split(",")]:
        x = torch.randn(B, d, device="cuda", generator=g)
        row = {"B": B}
        for mode in args.modes.split(","):
            os.environ["HIRE_UNION"] = mode
            with torch.cuda.stream(s):
                for f, a in layers:
                    H.ffn_group_sparse(f, x, a, k, kp, x_mode=H.X_INT8)
                s.synchronize()
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=s):
                    for i in range(20):
                        f, a = layers[i % 4]
                        H.ffn_group_sparse(f, x, a, k, kp, x_mode=H.X_INT8)
                for _ in range(3):
                    gr.replay()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(5):
                    gr.replay()
                e1.record(s)
                s.synchronize()
                row["union" if mode == "1" else "per_query"] = round(e0.elapsed_time(e1) * 1e3 / 100, 2)
        print(json.dumps(row))


if __name__ == "__main__":
    main()
