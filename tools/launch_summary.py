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
        agg.setdefault(short, []).append(float(r[iv]) / 1e3)
    # a launch far above its kernel's median is another use of the kernel in
    # the same command (the recall check's dense exact pass runs recompute_fast
    # over every row): listed, not counted in the step shares
    other = []
    for k, v in agg.items():
        med = sorted(v)[len(v) // 2]
        other += [(k, t) for t in v if t > 5 * med]
        agg[k] = [t for t in v if t <= 5 * med]
    tot = sum(sum(v) for v in agg.values()) or 1.0
    print(f"# {path}: our per-step kernels from the ncu launch list (--metrics gpu__time_duration.sum --clock-control none;")
    print("# serialised and cold-cache: use the shares, not the absolutes). One-time proxy build kernels excluded.")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:52s} launches {len(v):4d}  avg {sum(v) / len(v):8.2f} us  share {100 * sum(v) / tot:5.1f}%")
    for k, t in other:
        print(f"# not a step launch: {k} {t:.1f} us (dense exact pass of the recall check)")


if __name__ == "__main__":
    main(sys.argv[1])
