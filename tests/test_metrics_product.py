"""The product's recall and cost model (api.recall / param_bytes /
roofline_bytes, include/hire_b200.hpp hire::recall / hire::param_bytes)
pinned to the reference's own known answers: test_metrics.cpp:29-53
(recall set arithmetic) and :72-104 (param_bytes worked example and edge
cases), metrics.hpp:23-64. Host arithmetic only (no GPU)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def A():
    from paper_2402_09360_b200 import api
    return api


@pytest.mark.parametrize("cand,exact,want", [
    ([1, 2, 3, 4], [2, 5], (0.5, 1, True)),            # SetArithmetic
    ([0, 1, 2, 3, 4, 5], [4, 1, 5], (1.0, 3, True)),   # FullContainment
    ([1, 3], [0, 1], (0.5, 1, False)),                 # MissedTopOne
    ([1, 2], [], (0.0, 0, False)),                     # empty exact set (metrics.hpp:26)
])
def test_recall_matches_reference_cases(A, cand, exact, want):
    assert A.recall(np.array(cand, dtype=np.uint32), np.array(exact, dtype=np.uint32)) == want


def test_param_bytes_worked_example(A):
    c = A.param_bytes(100, 1000, 10, 50)
    assert (c.bytes_baseline, c.bytes_lr, c.bytes_q) == (200000, 32000, 60000)
    assert not c.lr_no_saving and not c.q_no_saving


def test_param_bytes_edge_cases(A):
    c = A.param_bytes(16, 64, 4, 0)
    assert c.bytes_lr == 2 * (16 * 4 + 4 * 64) and c.bytes_q == 16 * 64 // 2
    c = A.param_bytes(8, 32, 8, 32)
    assert c.bytes_lr == 2 * (8 * 8 + 8 * 32 + 8 * 32) and c.bytes_lr >= c.bytes_baseline and c.lr_no_saving
    assert A.param_bytes(3, 5, 1, 2).bytes_q == (3 * 5 + 1) // 2 + 2 * 3 * 2
    with pytest.raises(ValueError, match="param_bytes: dims must be positive"):
        A.param_bytes(0, 5, 1, 2)


def test_param_bytes_matches_oracle(A):
    import oracle as O
    for d, l, r, kp in [(100, 1000, 10, 50), (3, 5, 1, 2), (2048, 256000, 64, 1024)]:
        want = O.param_bytes(d, l, r, kp)
        got = A.param_bytes(d, l, r, kp)
        assert (got.bytes_baseline, got.bytes_lr, got.bytes_q, got.bytes_lrq) == tuple(want[:4])


def test_roofline_bytes_cfg3_and_cfg2(A):
    # BASELINE.md §4 / SURVEY.md §8(d): cfg3 B=1 = 263,168,000 proxy + 1024 x 2048 x 2
    assert A.roofline_bytes("q4", 2048, 256000, 1024, 2048 * 2) == 263_168_000 + 4_194_304
    # cfg2 B=1: proxy 8,421,376 + 820 U rows + 410 V rows (bf16)
    assert A.roofline_bytes("q4", 2048, 8192, 820, 4096, extra_rows=410) == 8_421_376 + 3_358_720 + 1_679_360
    # cfg1: fp32 rank-64 factors 8,650,752 + 256 x 1024 x 4
    assert A.roofline_bytes("lowrank", 1024, 32768, 256, 4096, r=64, factor_bytes=4) == 8_650_752 + 1_048_576


def test_cpp_param_bytes_and_recall(tmp_path):
    """hire_b200.hpp's host-side metrics compile and give the reference's
    known answers (no device call)."""
    src = tmp_path / "m.cpp"
    src.write_text(r'''
#include "hire_b200.hpp"
#include <cstdio>
int main() {
  auto c = hire::param_bytes(100, 1000, 10, 50);
  if (c.bytes_baseline != 200000u || c.bytes_lr != 32000u || c.bytes_q != 60000u) return 1;
  if (hire::param_bytes(3, 5, 1, 2).bytes_q != (3u * 5 + 1) / 2 + 2u * 3 * 2) return 2;
  try { hire::param_bytes(0, 5, 1, 2); return 3; } catch (const std::invalid_argument& e) {
    if (std::string(e.what()) != "param_bytes: dims must be positive") return 4; }
  hire::CandidateSet cs; cs.indices = {1, 2, 3, 4};
  hire::TopKSet ex; ex.k = 2; ex.entries.push_back({2, 99.0f}); ex.entries.push_back({5, 98.0f});
  auto r = hire::recall(cs, ex);
  if (r.recall != 0.5 || r.intersection_k != 1 || !r.top1_agree) return 5;
  std::puts("ok");
  return 0;
}
''')
    exe = tmp_path / "m"
    cc = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
                         "/usr/local/cuda/include", str(src), "-o", str(exe),
                         "-L", os.path.join(ROOT, "paper_2402_09360_b200"), "-lhire_cuda",
                         "-Wl,-rpath," + os.path.join(ROOT, "paper_2402_09360_b200")],
                        capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr[-3000:]
    run = subprocess.run([str(exe)], capture_output=True, text=True)
    assert run.returncode == 0 and run.stdout.strip() == "ok", (run.returncode, run.stdout, run.stderr)
