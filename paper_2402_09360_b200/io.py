"""The reference's weight files straight into device handles (SURVEY.md §8 f,
rank 1): HIRM matrices (io.hpp:94-107), HIRQ int4 proxies
(approx.hpp:551-586), HIRL low-rank proxies (approx.hpp:588-608).

Byte layout (little-endian, the reference's put_u32/put_f32): a 4-byte magic,
u32 dimensions, then fp32 blocks / packed nibbles. A reference column
(d contiguous values) is one row of this repo's row-major device layout, so
HIRM and HIRQ payloads load without reordering; HIRL's z2 (l x r, column-
major) is transposed into the [l][r] coefficient rows the kernels read.
Errors mirror the reference's IoError messages ("io: bad magic, expected
HIRM", "io: truncated ...", "io: cannot open for read: <path>")."""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as L


class HireIoError(L.HireError, OSError):
    """The reference's hire::IoError."""

    def __init__(self, msg: str):
        super().__init__(L.ERR_IO, msg)


def _read(path: str) -> bytes:
    try:
        with open(path, "rb") as fh:
            return fh.read()
    except OSError:
        raise HireIoError(f"io: cannot open for read: {path}") from None


class _Reader:
    def __init__(self, buf: bytes):
        self.b, self.o = buf, 0

    def magic(self, m: str):
        if self.b[self.o:self.o + 4] != m.encode():
            raise HireIoError(f"io: bad magic, expected {m}")
        self.o += 4

    def u32(self) -> int:
        if self.o + 4 > len(self.b):
            raise HireIoError("io: truncated file (u32)")
        v = int.from_bytes(self.b[self.o:self.o + 4], "little")
        self.o += 4
        return v

    def f32(self, n: int) -> np.ndarray:
        if self.o + 4 * n > len(self.b):
            raise HireIoError("io: truncated file (f32)")
        a = np.frombuffer(self.b, dtype="<f4", count=n, offset=self.o).astype(np.float32)
        self.o += 4 * n
        return a

    def raw(self, n: int, what: str) -> np.ndarray:
        if self.o + n > len(self.b):
            raise HireIoError(f"io: truncated {what} payload")
        a = np.frombuffer(self.b, dtype=np.uint8, count=n, offset=self.o)
        self.o += n
        return a


# ---- parsers (host, no device) ------------------------------------------
def parse_matrix(buf: bytes):
    """HIRM -> (rows d, cols l, values [l][d] float32)."""
    r = _Reader(buf)
    r.magic("HIRM")
    rows, cols = r.u32(), r.u32()
    return rows, cols, r.f32(rows * cols).reshape(cols, rows)


def parse_quantized(buf: bytes):
    """HIRQ -> (rows d, cols l, packed payload bytes, scales [l])."""
    r = _Reader(buf)
    r.magic("HIRQ")
    rows, cols = r.u32(), r.u32()
    scales = r.f32(cols)
    payload = r.raw((rows * cols + 1) // 2, "HIRQ")
    return rows, cols, payload, scales


def parse_low_rank(buf: bytes):
    """HIRL -> (z1 [r][d], z2 [l][r]) float32 in the device layouts."""
    r = _Reader(buf)
    r.magic("HIRL")
    d, l, rank = r.u32(), r.u32(), r.u32()
    z1 = r.f32(d * rank).reshape(rank, d)        # column q of the d x r matrix = row q
    z2 = r.f32(l * rank).reshape(rank, l).T      # l x r column-major -> [l][r]
    return np.ascontiguousarray(z1), np.ascontiguousarray(z2)


# ---- writers (the reference's byte layout; for tools and tests) ----------
def format_matrix(values_ld: np.ndarray) -> bytes:
    v = np.ascontiguousarray(values_ld, dtype="<f4")
    l, d = v.shape
    return b"HIRM" + d.to_bytes(4, "little") + l.to_bytes(4, "little") + v.tobytes()


def format_low_rank(z1_rd: np.ndarray, z2_lr: np.ndarray) -> bytes:
    z1 = np.ascontiguousarray(z1_rd, dtype="<f4")
    z2 = np.ascontiguousarray(np.asarray(z2_lr, dtype="<f4").T)
    r, d = z1.shape
    l = z2.shape[1]
    return (b"HIRL" + d.to_bytes(4, "little") + l.to_bytes(4, "little") + r.to_bytes(4, "little") +
            z1.tobytes() + z2.tobytes())


# ---- loaders into device handles ------------------------------------------
def read_matrix_file(path: str, dtype=torch.float32):
    """io.hpp:109-112 read_matrix_file -> ScoreMatrix on the device
    (dtype bfloat16: round-to-nearest-even, approx.hpp:76-81)."""
    from .api import ScoreMatrix
    _, _, vals = parse_matrix(_read(path))
    return ScoreMatrix(torch.from_numpy(vals).cuda().to(dtype))


def read_quantized_file(path: str):
    """approx.hpp:566-586 read_quantized -> int4 ApproxScorer (device layout
    built from the packed payload as is)."""
    from .api import ApproxScorer
    d, l, payload, scales = parse_quantized(_read(path))
    return ApproxScorer.from_hirq(payload, scales, l, d)


def read_low_rank_file(path: str, dtype=torch.float32):
    """approx.hpp:597-608 read_low_rank -> low-rank ApproxScorer."""
    from .api import ApproxScorer
    z1, z2 = parse_low_rank(_read(path))
    return ApproxScorer.low_rank(torch.from_numpy(z1).cuda().to(dtype), torch.from_numpy(z2).cuda().to(dtype))
