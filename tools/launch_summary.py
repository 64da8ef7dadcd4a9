"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, average durations and shares of our kernels' time
(the one-time proxy build / layout kernels and torch kernels excluded).

  python tools/launch_summary.py profiles/<run>.csv > profiles/<run>_summary.txt
"""
import collections
import csv
import sys

ONE_TIME = ("quantize_q4_kernel", "q4_to_mma_layout", "q4_to_umma_layout")
OURS = ("q4_", "sel_", "recompute", "final", "prep_x", "lr_", "ffn_", "fetch_host", "add_offset", "bucket_",
        "select_candidates", "gather_values", "group_", "expand_", "iota", "concat_sel", "sum_parts")


def main(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ik]
        base = name.replace("void ", "").replace("hire_dev::", "")
        if "hire_dev::" not in name and not base.startswith(OURS):
            continue
        if any(o in name for o in ONE_TIME):
            continue
        short = name.split("(")[0].replace("void ", "")
        n, t = agg.get(short, (0, 0.0))
        agg[short] = (n + 1, t + float(r[iv]) / 1e3)
    tot = sum(t for _, t in agg.values()) or 1.0
    print(f"# {path}: our per-step kernels from the ncu launch list (--metrics gpu__time_duration.sum --clock-control none;")
    print("# serialised and cold-cache: use the shares, not the absolutes). One-time proxy build kernels excluded.")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:52s} launches {n:4d}  avg {t / n:8.2f} us  share {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
