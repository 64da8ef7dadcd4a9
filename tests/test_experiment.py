"""The experiment runner (paper_2402_09360_b200/experiment.py, the
reference's experiment.hpp modes on the GPU path).

CPU: the library's host generators (Rng / derive_seed / gen_vector /
gen_instance, rng.hpp + instance.hpp) give the compiled reference's bits;
config parsing and its errors follow experiment.hpp (field names, messages,
exit codes). GPU: the mode rows equal the compiled reference on the same
seeded instance (strict fp32-x int4 scorer -> identical top-k rows and
values), and every mode runs and writes the reference's CSV layout."""
import json
import os

import numpy as np
import pytest


@pytest.fixture(scope="module")
def E():
    from paper_2402_09360_b200 import experiment
    return experiment


def _ref(O):
    if not O.ref_available():
        pytest.skip("compiled reference not built")
    return O.ref()


def test_generators_match_reference(E, O):
    R = _ref(O)
    import ctypes as C
    for seed, stream in [(0, 1), (7, 2), (123456789, 10000), (2 ** 63 + 5, 100)]:
        assert E.derive_seed(seed, stream) == R.ref_derive_seed(seed, stream)
    for dim, seed in [(1, 3), (64, 11), (1001, 99)]:
        want = np.empty(dim, np.float32)
        R.ref_gen_vector(dim, seed, want.ctypes.data_as(C.c_void_p))
        assert np.array_equal(E.gen_vector(dim, seed).view(np.uint32), want.view(np.uint32))
    for d, l, seed, dec in [(8, 30, 5, False), (16, 40, 6, True), (33, 7, 9, True)]:
        want = np.empty((l, d), np.float32)
        assert R.ref_gen_instance(d, l, seed, int(dec), want.ctypes.data_as(C.c_void_p)) == 0
        assert np.array_equal(E.gen_instance(d, l, seed, dec).view(np.uint32), want.view(np.uint32)), (d, l, dec)


def test_config_parsing_and_errors(E, tmp_path):
    c = E.parse_config({"mode": "cost", "d": 100, "l": 1000, "rank": 10, "k_prime": [50, 60], "seed": 3})
    assert (c.mode, c.d, c.l, c.rank, c.k_prime, c.seed) == ("cost", 100, 1000, 10, [50, 60], 3)
    assert E.parse_config({"k_prime": 7}).k_prime == [7]
    for bad, fld in [({"d": -1}, "d"), ({"nope": 1}, "nope"), ({"k_prime": []}, "k_prime"), ({"scorer": 3}, "scorer")]:
        with pytest.raises(E.ConfigError, match=f"field '{fld}'"):
            E.parse_config(bad)
    # cost mode needs no GPU: the reference's worked example (test_metrics.cpp:72-80)
    out = tmp_path / "cost.csv"
    rc = E.main(["--mode", "cost", "--d", "100", "--l", "1000", "--rank", "10", "--k_prime", "50", "--out", str(out)])
    assert rc == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "# mode=cost seed=0 d=100 l=1000 m=512 g=8 k=32 scorer=quantized version=0.1.0"
    assert lines[1:] == ["method,bytes", "baseline,200000", "lr,32000", "q,60000", "lrq," + str((100 * 10 + 10 * 1000 + 1) // 2 + 2 * 100 * 50)]
    assert E.main(["--mode", "nonsense", "--out", str(tmp_path / "x.csv")]) == 1
    assert not (tmp_path / "x.csv").exists()  # no partial artifact
    assert E.main(["--mode", "cost"]) == 1  # out required
    cfgf = tmp_path / "bad.json"
    cfgf.write_text("{not json")
    assert E.main(["--config", str(cfgf)]) == 1
    assert E.main(["--config", str(tmp_path / "missing.json")]) == 2


@pytest.mark.gpu
def test_hire_and_softmax_and_distributed_rows_equal_reference(E, O, tmp_path):
    R = _ref(O)
    base = ["--d", "64", "--l", "1024", "--k", "16", "--k_prime", "64", "--seed", "5"]
    rows = {}
    for mode in ("hire-topk", "softmax-topk", "distributed"):
        out = tmp_path / f"{mode}.csv"
        assert E.main(["--mode", mode, *base, "--shards", "4", "--out", str(out)]) == 0
        rows[mode] = [l for l in out.read_text().splitlines() if not l.startswith("#")][1:]
    w = E.gen_instance(64, 1024, E.derive_seed(5, 1))
    x = E.gen_vector(64, E.derive_seed(5, 2))
    codes, scales = O.ref_quantize_int4(w)
    rm, ra = O.RefMatrix(w), O.RefScorer("quantized", codes=codes, scales=scales)
    r = O.ref_hire_topk(rm, ra, x, 16, 64)
    assert rows["hire-topk"] == [f"{i},{j},{E.fmt_real(v)}" for i, (j, v) in enumerate(zip(r["top_idx"], r["top_val"]))]
    idx, pr = O.ref_softmax_topk(rm, ra, x, 16, 64)
    got = [l.split(",") for l in rows["softmax-topk"]]
    assert [int(g[1]) for g in got] == list(map(int, idx))
    np.testing.assert_allclose([float(g[2]) for g in got], pr, rtol=1e-6)
    ti, tv, _, _ = O.ref_da_topk(rm, ra, x, 4, 16, 64)
    assert rows["distributed"] == [f"{i},{j},{E.fmt_real(v)}" for i, (j, v) in enumerate(zip(ti, tv))]


@pytest.mark.gpu
def test_every_mode_runs(E, tmp_path):
    runs = {
        "ffn": ["--d", "64", "--m", "512", "--g", "8", "--k", "64", "--k_prime", "128", "--m1", "64"],
        "kprime-sweep": ["--d", "32", "--l", "512", "--k", "8", "--k_prime", "8,16,64,512", "--n_samples", "3"],
        "overlap": ["--d", "32", "--m", "256", "--g", "4", "--k", "32", "--k_prime", "64", "--trials", "3", "--n_samples", "4"],
        "bench-gather": ["--d", "128", "--n_groups", "512", "--g", "8", "--g_sweep", "1,8,64", "--repeats", "3"],
        "gen-instance": ["--d", "16", "--l", "40", "--matrix_file", str(tmp_path / "z.hirm"),
                         "--vector_file", str(tmp_path / "x.hirv"), "--instance", "random-decaying"],
    }
    for mode, args in runs.items():
        out = tmp_path / f"{mode}.csv"
        assert E.main(["--mode", mode, *args, "--out", str(out)]) == 0, mode
        lines = out.read_text().splitlines()
        assert lines[0].startswith(f"# mode={mode} ")
    ffn = (tmp_path / "ffn.csv").read_text().splitlines()
    assert [l.split(",")[0] for l in ffn[1:]] == ["variant", "dense", "topk", "group-sparse", "common-path"]
    ks = (tmp_path / "kprime-sweep.csv").read_text().splitlines()
    rec = [float(l.split(",")[1]) for l in ks[2:]]
    assert rec == sorted(rec) and rec[-1] == 1.0  # monotone in k' (acceptance_test.cpp:146-177); k' = all -> 1
    # a generated instance file feeds instance=file back in
    out = tmp_path / "file.csv"
    assert E.main(["--mode", "hire-topk", "--instance", "file", "--matrix_file", str(tmp_path / "z.hirm"),
                   "--vector_file", str(tmp_path / "x.hirv"), "--k", "4", "--k_prime", "8", "--out", str(out)]) == 0
    assert E.main(["--mode", "projection-ablation", "--out", str(tmp_path / "p.csv")]) == 1
