"""FMV1 vector persistence (SPEC.md cli module save_vector / load_vector;
SURVEY.md §8 f4) -- the Python mirror of include/fftmv/vector_io.hpp, byte
for byte: "FMV1", little-endian u64 space_extent, time_extent, layout code
(0 SOTI, 1 TOSI), precision code (0 f64, 1 f32), domain code (0 time,
1 frequency), then the raw little-endian scalars. load(save(v)) is bitwise."""
from __future__ import annotations

import struct

import numpy as np

from .fftmv import BlockVector, Domain, Layout, Precision

__all__ = ["encode_vector", "decode_vector", "save_vector", "load_vector"]

_HDR = struct.Struct("<4s5Q")


def encode_vector(v: BlockVector) -> bytes:
    if v.precision not in (Precision.Double, Precision.Single):
        raise ValueError("FMV1: fp16 vectors have no precision code")
    v.validate()
    dt = "<f8" if v.precision == Precision.Double else "<f4"
    data = np.ascontiguousarray(v.data, dtype=dt)
    hdr = _HDR.pack(b"FMV1", v.space_extent, v.time_extent, 0 if v.layout == Layout.SOTI else 1,
                    0 if v.precision == Precision.Double else 1, 0 if v.domain == Domain.Time else 1)
    return hdr + data.tobytes()


def decode_vector(b: bytes) -> BlockVector:
    if len(b) < 4 or b[:4] != b"FMV1":
        raise ValueError("FMV1: bad magic")
    if len(b) < _HDR.size:
        raise ValueError("FMV1: truncated file (header)")
    _, s, t, lay, prec, dom = _HDR.unpack_from(b)
    for name, code in (("layout", lay), ("precision", prec), ("domain", dom)):
        if code > 1:
            raise ValueError(f"FMV1: {name} code out of range ({code})")
    es = 8 if prec == 0 else 4
    scalars = s * t * (2 if dom == 1 else 1)
    have = len(b) - _HDR.size
    if s == 0 or t == 0 or have != scalars * es:
        raise ValueError(f"FMV1: truncated/oversized payload ({have} bytes for {scalars} scalars of {es} bytes)")
    data = np.frombuffer(b, dtype="<f8" if prec == 0 else "<f4", offset=_HDR.size).astype(
        np.float64 if prec == 0 else np.float32)
    return BlockVector(s, t, Layout.SOTI if lay == 0 else Layout.TOSI,
                       Precision.Double if prec == 0 else Precision.Single,
                       Domain.Time if dom == 0 else Domain.Frequency, data)


def save_vector(path: str, v: BlockVector) -> None:
    with open(path, "wb") as f:
        f.write(encode_vector(v))


def load_vector(path: str) -> BlockVector:
    with open(path, "rb") as f:
        return decode_vector(f.read())
