"""The reference's experiment runner (experiment.hpp:28-652, the `hire` CLI's
config-driven modes) driving the B200 path.

    python -m paper_2402_09360_b200.experiment --mode hire-topk --d 64 --l 1024 --k 32 --k_prime 64 --out r.csv
    python -m paper_2402_09360_b200.experiment --config exp.json [--field value ...]

Same config fields and defaults (ExperimentConfig, experiment.hpp:55-84), the
same seeded instances (gen_instance / gen_vector / derive_seed through the
library's host generators, bit-identical to the reference's), the same CSV
artifacts (manifest line, columns, "%.9g" reals, written on close) and exit
codes (0 ok, 1 config, 2 I/O, 3 numeric). The scorer runs in strict mode
(fp32 x, the reference's summation order), so the rows equal the reference's.

Modes: hire-topk, softmax-topk, distributed (DA-TOP-k over `shards`), ffn
(dense / top-k / group-sparse / common-path), kprime-sweep, overlap,
bench-gather (GPU gather microbenchmark), cost, gen-instance. Not built:
projection-ablation and the low-rank scorers, which need the offline SVD /
random-projection fits (fit_low_rank_svd, random_low_rank — DESIGN.md "Out of
scope"); scorer "exact" (exact_copy) likewise.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys
from dataclasses import dataclass, field
from typing import List

import numpy as np
import torch

from . import _lib as L
from . import api as A
from ._lib import check, lib

VERSION = "0.1.0"
EXIT_OK, EXIT_CONFIG, EXIT_IO, EXIT_NUMERIC = 0, 1, 2, 3


class ConfigError(Exception):
    """experiment.hpp:36-40."""

    def __init__(self, field_name: str, what: str):
        super().__init__(f"config error: field '{field_name}': {what}")
        self.field_name = field_name


class IoError(Exception):
    pass


class NumericError(Exception):
    pass


@dataclass
class ExperimentConfig:
    """experiment.hpp:55-84 (field names, defaults)."""
    mode: str = ""
    d: int = 64
    l: int = 1024
    m: int = 512
    g: int = 8
    m1: int = 0
    m2: int = 0
    k: int = 32
    k_prime: List[int] = field(default_factory=lambda: [64])
    rank: int = 8
    scorer: str = "quantized"
    shards: int = 2
    n_samples: int = 8
    trials: int = 100
    seed: int = 0
    instance: str = "random-gaussian"
    matrix_file: str = ""
    vector_file: str = ""
    ffn_file: str = ""
    out: str = ""
    phi: str = ""
    rho: float = 0.9
    n_groups: int = 2048
    fraction_selected: float = 0.25
    repeats: int = 9
    g_sweep: List[int] = field(default_factory=lambda: [1, 2, 4, 8, 16, 32, 64])


_COUNT = {"d", "l", "m", "g", "m1", "m2", "k", "rank", "shards", "n_samples", "trials", "n_groups", "repeats"}
_LIST = {"k_prime", "g_sweep"}
_STR = {"mode", "scorer", "instance", "matrix_file", "vector_file", "ffn_file", "out", "phi"}
_REAL = {"rho", "fraction_selected"}


def _as_count(v, key):
    if isinstance(v, bool) or not isinstance(v, int) or v < 0:
        raise ConfigError(key, "expected a non-negative integer")
    return v


def parse_config(obj: dict, cfg: ExperimentConfig = None) -> ExperimentConfig:
    """parse_config_json (experiment.hpp:118-167)."""
    cfg = cfg or ExperimentConfig()
    if not isinstance(obj, dict):
        raise ConfigError("config", "expected a JSON object")
    for key, value in obj.items():
        if key in _COUNT:
            setattr(cfg, key, _as_count(value, key))
        elif key in _LIST:
            if isinstance(value, list):
                if not value:
                    raise ConfigError(key, "sweep list must be non-empty")
                setattr(cfg, key, [_as_count(v, key) for v in value])
            else:
                setattr(cfg, key, [_as_count(value, key)])
        elif key in _STR:
            if not isinstance(value, str):
                raise ConfigError(key, "expected a string")
            setattr(cfg, key, value)
        elif key in _REAL:
            if isinstance(value, bool) or not isinstance(value, (int, float)):
                raise ConfigError(key, "expected a number")
            setattr(cfg, key, float(value))
        elif key == "seed":
            cfg.seed = _as_count(value, key)
        else:
            raise ConfigError(key, "unknown field")
    return cfg


def load_config_file(path: str) -> ExperimentConfig:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise IoError(f"io: cannot open config: {path}")
    try:
        obj = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError("config", f"invalid JSON: {e}")
    return parse_config(obj)


# ---- instances (instance.hpp through the library's host generators) -------
def derive_seed(seed: int, stream: int) -> int:
    return int(lib().hire_derive_seed(seed, stream))


def gen_vector(dim: int, seed: int) -> np.ndarray:
    out = np.empty(dim, dtype=np.float32)
    check(lib().hire_gen_vector(seed, dim, out.ctypes.data_as(C.c_void_p)))
    return out


def gen_instance(d: int, l: int, seed: int, decaying: bool = False) -> np.ndarray:
    """[l][d] (= the reference's d x l column-major ScoreMatrix)."""
    out = np.empty((l, d), dtype=np.float32)
    check(lib().hire_gen_instance(d, l, seed, 1 if decaying else 0, out.ctypes.data_as(C.c_void_p)))
    return out


def fmt_real(v: float) -> str:
    return "%.9g" % float(v)


class CsvWriter:
    """experiment.hpp:208-242: buffered, written on close."""

    def __init__(self, path: str):
        self.path, self.lines = path, []

    def manifest(self, c: ExperimentConfig):
        self.lines.append(f"# mode={c.mode} seed={c.seed} d={c.d} l={c.l} m={c.m} g={c.g} k={c.k} "
                          f"scorer={c.scorer} version={VERSION}")

    def comment(self, line: str):
        self.lines.append("# " + line)

    def row(self, fields):
        self.lines.append(",".join(str(f) for f in fields))

    def close(self):
        try:
            with open(self.path, "w", newline="") as f:
                f.write("\n".join(self.lines) + "\n")
        except OSError:
            raise IoError(f"io: cannot open for write: {self.path}")


def _phi(c: ExperimentConfig, default: str) -> str:
    name = c.phi or default
    if name not in ("identity", "relu", "squared-relu"):
        raise ConfigError("phi", f"expected identity | relu | squared-relu, got '{name}'")
    return name


def _require(ok: bool, fld: str, what: str):
    if not ok:
        raise ConfigError(fld, what)


def _T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _scorer(c: ExperimentConfig, w: np.ndarray):
    """build_scorer (experiment.hpp:190-205): the int4 proxy on the device."""
    if c.scorer == "quantized":
        return A.ApproxScorer.quantize(A.ScoreMatrix(_T(w)))
    if c.scorer in ("exact", "low-rank", "low-rank-quantized", "random-low-rank"):
        raise ConfigError("scorer", f"scorer '{c.scorer}' needs an offline proxy fit (not on the GPU path); "
                                    "use quantized")
    raise ConfigError("scorer", "expected exact | quantized | low-rank | low-rank-quantized | random-low-rank, "
                                f"got '{c.scorer}'")


def _read_hirv(path: str) -> np.ndarray:
    try:
        buf = open(path, "rb").read()
    except OSError:
        raise IoError(f"io: cannot open for read: {path}")
    if buf[:4] != b"HIRV" or len(buf) < 8:
        raise IoError(f"io: bad magic in {path}")
    n = int.from_bytes(buf[4:8], "little")
    return np.frombuffer(buf[8:8 + 4 * n], dtype="<f4").astype(np.float32)


def _instance(c: ExperimentConfig):
    """load_or_generate (experiment.hpp:250-275)."""
    if c.instance == "file":
        _require(bool(c.matrix_file), "matrix_file", "required when instance=file")
        _require(bool(c.vector_file), "vector_file", "required when instance=file")
        from .io import _read, parse_matrix
        _, _, w = parse_matrix(_read(c.matrix_file))
        x = _read_hirv(c.vector_file)
        if x.size != w.shape[1]:
            raise ConfigError("vector_file", f"vector dim {x.size} does not match matrix rows {w.shape[1]}")
        return np.ascontiguousarray(w, dtype=np.float32), x
    if c.instance not in ("random-gaussian", "random-decaying"):
        raise ConfigError("instance", f"expected random-gaussian | random-decaying | file, got '{c.instance}'")
    return (gen_instance(c.d, c.l, derive_seed(c.seed, 1), c.instance == "random-decaying"),
            gen_vector(c.d, derive_seed(c.seed, 2)))


def _strict(k, kp, phi="identity"):
    return A.HireConfig(k=k, k_prime=kp, phi=phi, strict=True)


# ---- modes ----------------------------------------------------------------
def run_hire_topk(c: ExperimentConfig, csv: CsvWriter):
    _require(bool(c.k_prime), "k_prime", "required")
    w, x = _instance(c)
    a = _scorer(c, w)
    r = A.hire_topk(_T(x[None]), A.ScoreMatrix(_T(w)), a, _strict(c.k, c.k_prime[0], _phi(c, "identity")))
    csv.row(["pos", "index", "value"])
    for i, (j, v) in enumerate(zip(r.top_idx[0].tolist(), r.top_val[0].tolist())):
        csv.row([i, j, fmt_real(v)])


def run_softmax_topk(c: ExperimentConfig, csv: CsvWriter):
    _require(bool(c.k_prime), "k_prime", "required")
    _require(c.phi in ("", "identity"), "phi", "softmax-topk requires identity")
    w, x = _instance(c)
    a = _scorer(c, w)
    idx, prob = A.softmax_topk(A.ScoreMatrix(_T(w)), _T(x[None]), a, _strict(c.k, c.k_prime[0]))
    csv.row(["pos", "index", "probability"])
    for i, (j, p) in enumerate(zip(idx[0].tolist(), prob[0].tolist())):
        csv.row([i, j, fmt_real(p)])


def run_distributed(c: ExperimentConfig, csv: CsvWriter):
    _require(bool(c.k_prime), "k_prime", "required")
    _require(c.shards >= 1, "shards", "must be >= 1")
    _require(c.k % c.shards == 0, "k", "shards must divide k for DA-TOP-k")
    _require(c.k_prime[0] % c.shards == 0, "k_prime", "shards must divide k_prime for DA-TOP-k")
    w, x = _instance(c)
    a = _scorer(c, w)
    l, d = w.shape
    ti, tv, _ = A.da_topk_emulated(A.ScoreMatrix(_T(w)), a, _T(x[None]), c.shards,
                                   _strict(c.k, c.k_prime[0], _phi(c, "identity")))
    # CommReport (distributed.hpp:121-124): per-shard candidates, 4 bytes per entry
    per = [min(c.k_prime[0] // c.shards, A.shard_range(l, c.shards, s)[1]) for s in range(c.shards)]
    csv.comment(f"shards={c.shards} bytes_gathered={sum(per) * d * 4} candidates_per_shard=" +
                "|".join(str(p) for p in per))
    csv.row(["pos", "index", "value"])
    for i, (j, v) in enumerate(zip(ti[0].tolist(), tv[0].tolist())):
        csv.row([i, j, fmt_real(v)])


def _rel_l2(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    num, den = float(((got - want) ** 2).sum()), float((want ** 2).sum())
    return math.sqrt(num / den) if den > 0 else math.sqrt(num)


def _l2(v):
    return math.sqrt(float((np.asarray(v, np.float64) ** 2).sum()))


def run_ffn(c: ExperimentConfig, csv: CsvWriter):
    _require(bool(c.k_prime), "k_prime", "required")
    phi = _phi(c, "relu")
    if c.instance == "file":
        _require(bool(c.ffn_file), "ffn_file", "required when instance=file")
        _require(bool(c.vector_file), "vector_file", "required when instance=file")
        try:
            buf = open(c.ffn_file, "rb").read()
        except OSError:
            raise IoError(f"io: cannot open for read: {c.ffn_file}")
        if buf[:4] != b"HIRF":
            raise IoError(f"io: bad magic in {c.ffn_file}")
        d, m, g = (int.from_bytes(buf[4 + 4 * i:8 + 4 * i], "little") for i in range(3))
        body = np.frombuffer(buf[20:20 + 8 * d * m], dtype="<f4")
        u, v = body[:d * m].reshape(m, d).copy(), body[d * m:].reshape(m, d).copy()
        x = _read_hirv(c.vector_file)
    else:
        u = gen_instance(c.d, c.m, derive_seed(c.seed, 1))
        v = gen_instance(c.d, c.m, derive_seed(c.seed, 2))
        g = c.g
        x = gen_vector(c.d, derive_seed(c.seed, 3))
    m = u.shape[0]
    _require(g >= 1 and m % g == 0, "g", "g must divide m")
    kp = c.k_prime[0]
    _require(1 <= c.k <= m, "k", "must be in [1, m]")
    _require(c.k % g == 0, "k", "g must divide k")
    _require(kp % g == 0, "k_prime", "g must divide k_prime")
    _require(c.k <= kp <= m, "k_prime", "need k <= k_prime <= m")
    U, V = A.ScoreMatrix(_T(u)), A.ScoreMatrix(_T(v))
    f = A.GroupedFFN(U, V, g, phi)
    a = _scorer(c, u)
    xt = _T(x[None])
    dense = A.ffn_dense(f, xt, strict=True)[0].cpu().numpy()
    # ffn_topk (ffn.hpp:78-100): the exact top-k units = group-sparse over
    # g = 1 with every unit a candidate
    topk, _ = A.ffn_group_sparse(A.GroupedFFN(U, V, 1, phi), xt, a, c.k, m, strict=True)
    gs, _ = A.ffn_group_sparse(f, xt, a, c.k, kp, strict=True)
    topk, gs = topk[0].cpu().numpy(), gs[0].cpu().numpy()
    csv.row(["variant", "output_l2", "rel_err_vs_dense"])
    csv.row(["dense", fmt_real(_l2(dense)), fmt_real(0.0)])
    csv.row(["topk", fmt_real(_l2(topk)), fmt_real(_rel_l2(topk, dense))])
    csv.row(["group-sparse", fmt_real(_l2(gs)), fmt_real(_rel_l2(gs, dense))])
    if c.m1 > 0:
        m2 = m - c.m1
        _require(c.m2 == 0 or c.m2 == m2, "m2", "common path splits m, so m2 must equal m - m1")
        _require(c.m1 < m, "m1", "must be < m")
        _require(m2 % g == 0 and m2 >= g, "m1", "m - m1 must be a positive multiple of g")
        _require(c.k <= m2 and kp <= m2, "m1", "k and k_prime must fit the sparse part")
        cp = A.CommonPathFFN(A.GroupedFFN(U.slice_cols(0, c.m1), V.slice_cols(0, c.m1), 1, phi),
                             A.GroupedFFN(U.slice_cols(c.m1, m2), V.slice_cols(c.m1, m2), g, phi))
        out = A.ffn_common_path(cp, xt, a.slice_cols(c.m1, m2), c.k, kp, strict=True)[0].cpu().numpy()
        csv.row(["common-path", fmt_real(_l2(out)), fmt_real(_rel_l2(out, dense))])


def run_kprime_sweep(c: ExperimentConfig, csv: CsvWriter):
    _require(bool(c.k_prime), "k_prime", "required")
    _require(c.n_samples >= 1, "n_samples", "must be >= 1")
    phi = _phi(c, "identity")
    csv.row(["k_prime", "recall", "intersection_k", "top1_agree"])
    rec = np.zeros(len(c.k_prime))
    inter = np.zeros(len(c.k_prime))
    top1 = np.zeros(len(c.k_prime))
    for t in range(c.n_samples):
        w = gen_instance(c.d, c.l, derive_seed(c.seed, 100 + t))
        x = gen_vector(c.d, derive_seed(c.seed, 10000 + t))
        a = _scorer(c, w)
        z = A.ScoreMatrix(_T(w))
        ex, _, _ = A.exact_topk(z, _T(x[None]), c.k, phi, strict=True)
        exi = ex[0].cpu().numpy()
        for s, kp in enumerate(c.k_prime):
            r = A.hire_topk(_T(x[None]), z, a, _strict(c.k, kp, phi))
            rr, ik, t1 = A.recall(r.cand[0].cpu().numpy(), exi)
            rec[s] += rr
            inter[s] += ik
            top1[s] += 1.0 if t1 else 0.0
    n = float(c.n_samples)
    for s, kp in enumerate(c.k_prime):
        csv.row([kp, fmt_real(rec[s] / n), fmt_real(inter[s] / n), fmt_real(top1[s] / n)])


def run_overlap(c: ExperimentConfig, csv: CsvWriter):
    _require(bool(c.k_prime), "k_prime", "required")
    _require(c.n_samples >= 1, "n_samples", "must be >= 1")
    _require(c.trials >= 1, "trials", "must be >= 1")
    _require(0.0 <= c.rho <= 1.0, "rho", "must be in [0, 1]")
    phi = _phi(c, "relu")
    u = gen_instance(c.d, c.m, derive_seed(c.seed, 1))
    v = gen_instance(c.d, c.m, derive_seed(c.seed, 2))
    _require(c.g >= 1 and c.m % c.g == 0, "g", "g must divide m")
    kp = c.k_prime[0]
    _require(c.k % c.g == 0, "k", "g must divide k")
    _require(kp % c.g == 0, "k_prime", "g must divide k_prime")
    _require(c.k <= kp <= c.m, "k_prime", "need k <= k_prime <= m")
    f = A.GroupedFFN(A.ScoreMatrix(_T(u)), A.ScoreMatrix(_T(v)), c.g, phi)
    a = _scorer(c, u)
    noise = math.sqrt(max(0.0, 1.0 - c.rho * c.rho))
    csv.row(["trial", "union_groups", "overlap_ratio"])
    for t in range(c.trials):
        base = gen_vector(c.d, derive_seed(c.seed, 100 + t))
        xs = np.stack([gen_vector(c.d, derive_seed(c.seed, 10000 + t * 1024 + s)) for s in range(c.n_samples)])
        xs = (c.rho * base.astype(np.float64) + noise * xs.astype(np.float64)).astype(np.float32)
        _, sel = A.ffn_group_sparse(f, _T(xs), a, c.k, kp, strict=True)
        sets = [np.asarray(sorted(set(sel[s].tolist())), np.uint32) for s in range(c.n_samples)]
        union = len(set().union(*[set(s.tolist()) for s in sets]))
        csv.row([t, union, fmt_real(union / (c.n_samples * (c.k // c.g)))])


def run_bench_gather(c: ExperimentConfig, csv: CsvWriter):
    _require(bool(c.g_sweep), "g_sweep", "must be non-empty")
    units = c.n_groups * c.g
    csv.row(["g", "bytes", "sparse_ns", "dense_ns", "efficiency_paper", "efficiency_ratio"])
    for g in c.g_sweep:
        _require(g >= 1 and units % g == 0, "g_sweep", f"every g must divide n_groups*g = {units}")
        r = A.run_gather_bench(A.GatherBenchConfig(units // g, g, c.d, c.fraction_selected, c.repeats, c.seed))
        if not r.checksum_ok:
            raise NumericError(f"bench-gather: checksum mismatch at g = {g}")
        csv.row([g, r.bytes_moved, fmt_real(r.sparse_ns), fmt_real(r.dense_ns), fmt_real(r.efficiency_paper),
                 fmt_real(r.efficiency_ratio)])


def run_cost(c: ExperimentConfig, csv: CsvWriter):
    _require(bool(c.k_prime), "k_prime", "required")
    r = A.param_bytes(c.d, c.l, c.rank, c.k_prime[0])
    csv.row(["method", "bytes"])
    for name, v in (("baseline", r.bytes_baseline), ("lr", r.bytes_lr), ("q", r.bytes_q), ("lrq", r.bytes_lrq)):
        csv.row([name, v])


def run_gen_instance(c: ExperimentConfig, csv: CsvWriter):
    _require(bool(c.matrix_file), "matrix_file", "required")
    _require(bool(c.vector_file), "vector_file", "required")
    if c.instance not in ("random-gaussian", "random-decaying"):
        raise ConfigError("instance", "gen-instance needs random-gaussian | random-decaying")
    from .io import format_matrix
    w = gen_instance(c.d, c.l, derive_seed(c.seed, 1), c.instance == "random-decaying")
    x = gen_vector(c.d, derive_seed(c.seed, 2))
    try:
        with open(c.matrix_file, "wb") as f:
            f.write(format_matrix(w))
        with open(c.vector_file, "wb") as f:
            f.write(b"HIRV" + int(x.size).to_bytes(4, "little") + x.astype("<f4").tobytes())
    except OSError as e:
        raise IoError(f"io: write failed: {e.filename}")
    csv.row(["artifact", "path"])
    csv.row(["matrix", c.matrix_file])
    csv.row(["vector", c.vector_file])


MODES = {"hire-topk": run_hire_topk, "softmax-topk": run_softmax_topk, "distributed": run_distributed,
         "ffn": run_ffn, "kprime-sweep": run_kprime_sweep, "overlap": run_overlap,
         "bench-gather": run_bench_gather, "cost": run_cost, "gen-instance": run_gen_instance}


def run_experiment(c: ExperimentConfig):
    """run_experiment (experiment.hpp:607-630)."""
    if not c.mode:
        raise ConfigError("mode", "required")
    if not c.out:
        raise ConfigError("out", "required")
    csv = CsvWriter(c.out)
    csv.manifest(c)
    if c.mode == "projection-ablation":
        raise ConfigError("mode", "projection-ablation needs the offline SVD / random-projection fits "
                                  "(not on the GPU path)")
    fn = MODES.get(c.mode)
    if fn is None:
        raise ConfigError("mode", f"unknown mode '{c.mode}'")
    fn(c, csv)
    csv.close()


def run_experiment_catching(c: ExperimentConfig) -> int:
    """experiment.hpp:633-651: the error taxonomy -> exit codes."""
    try:
        run_experiment(c)
        return EXIT_OK
    except ConfigError as e:
        print(e, file=sys.stderr)
        return EXIT_CONFIG
    except L.HireInvalidArgument as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except IoError as e:
        print(e, file=sys.stderr)
        return EXIT_IO
    except (NumericError, L.HireError) as e:
        print(f"numeric error: {e}", file=sys.stderr)
        return EXIT_NUMERIC


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--config")
    args, rest = ap.parse_known_args(argv)
    try:
        cfg = load_config_file(args.config) if args.config else ExperimentConfig()
        # --field value flags override the file (values parsed as JSON when they can be)
        over = {}
        it = iter(rest)
        for flag in it:
            if not flag.startswith("--"):
                raise ConfigError(flag, "expected --field value")
            key = flag[2:].replace("-", "_")
            try:
                raw = next(it)
            except StopIteration:
                raise ConfigError(key, "missing value")
            try:
                val = json.loads(raw)
            except json.JSONDecodeError:
                val = raw
            if key in _STR:
                val = raw
            if key in _LIST and isinstance(val, str):
                val = [json.loads(p) for p in val.split(",")]
            over[key] = val
        cfg = parse_config(over, cfg)
    except ConfigError as e:
        print(e, file=sys.stderr)
        return EXIT_CONFIG
    except IoError as e:
        print(e, file=sys.stderr)
        return EXIT_IO
    return run_experiment_catching(cfg)


if __name__ == "__main__":
    sys.exit(main())
