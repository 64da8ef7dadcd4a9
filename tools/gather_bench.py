"""bench-gather mode of the reference's experiment runner
(experiment.hpp:547-572) on the GPU: one CSV row per group size g with the
reference's columns. Usage: python tools/gather_bench.py [n_groups*g] [d] [fraction] [g,g,...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_09360_b200 as H  # noqa: E402


def main():
    units = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
    frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
    sweep = [int(g) for g in (sys.argv[4] if len(sys.argv) > 4 else "1,2,4,8,16,32").split(",")]
    print("g,bytes,sparse_ns,dense_ns,efficiency_paper,efficiency_ratio")
    for g in sweep:
        if units % g:
            raise SystemExit(f"g_sweep: every g must divide n_groups*g = {units}")
        r = H.run_gather_bench(H.GatherBenchConfig(n_groups=units // g, g=g, d=d, fraction_selected=frac, repeats=9))
        if not r.checksum_ok:
            raise SystemExit(f"bench-gather: checksum mismatch at g = {g}")
        print(f"{g},{r.bytes_moved},{r.sparse_ns:.6g},{r.dense_ns:.6g},{r.efficiency_paper:.6g},{r.efficiency_ratio:.6g}")


if __name__ == "__main__":
    main()
