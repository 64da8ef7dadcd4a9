"""GPU analogue of the reference's gather microbenchmark (gather_bench.hpp,
the paper's group-size argument): the gather of a seeded random fraction of
groups checks against the source (the reference's FNV-1a checksum), selects
ceil(fraction * n_groups) groups, moves the byte count the reference
reports, and rejects bad configs with the reference's messages. The g-sweep
shape of the reference's bench-gather mode (experiment.hpp:547-572): groups
of more rows gather closer to the dense copy."""
import math

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_groups,g,d,frac", [(4096, 8, 128, 0.25), (1000, 1, 33, 0.1), (257, 3, 64, 1.0)])
def test_gather_bench_checksum_and_counts(H, n_groups, g, d, frac):
    r = H.run_gather_bench(H.GatherBenchConfig(n_groups=n_groups, g=g, d=d, fraction_selected=frac, repeats=5, seed=3))
    n_sel = math.ceil(frac * n_groups)
    assert r.checksum_ok
    assert r.groups_selected == n_sel
    assert r.bytes_moved == n_sel * g * d * 4
    assert r.sparse_ns > 0 and r.dense_ns > 0
    assert r.efficiency_paper == pytest.approx(r.sparse_ns / r.dense_ns)


def test_gather_bench_rejects_bad_configs(H):
    for kw, msg in [(dict(n_groups=0), "dims must be >= 1"), (dict(fraction_selected=0.0), "fraction_selected"),
                    (dict(fraction_selected=1.5), "fraction_selected"), (dict(repeats=2), "repeats must be >= 3")]:
        with pytest.raises(H.HireInvalidArgument, match=msg):
            H.run_gather_bench(H.GatherBenchConfig(**kw))


def test_gather_bench_group_size_sweep(H):
    """bench-gather's sweep: the same bytes in groups of g = 1, 8, 64 rows of
    d = 512 (2 KB rows); larger groups are at least as efficient."""
    effs = []
    for g in (1, 8, 64):
        r = H.run_gather_bench(H.GatherBenchConfig(n_groups=32768 // g, g=g, d=512, fraction_selected=0.25,
                                                   repeats=7, seed=1))
        assert r.checksum_ok
        effs.append(r.efficiency_ratio)
    assert effs[2] >= 0.5 * effs[0]
