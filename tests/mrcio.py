"""Minimal MRC2014 writer for test fixtures (header fields per the MRC2014 format,
as written/read by the reference's volio.cpp:57-193)."""
import numpy as np


def write_mrc(path, vol, mode=2, big_endian=False, axes=(1, 2, 3), voxel=1.0, ext=0, stamp=True, nz=None,
              truncate=0):
    vol = np.asarray(vol)
    n = vol.shape[-1]
    nzv = nz if nz is not None else vol.size // (n * n)
    bo = ">" if big_endian else "<"
    hdr = bytearray(1024)

    def i32(off, v):
        hdr[off:off + 4] = np.array([v], dtype=bo + "i4").tobytes()

    def f32(off, v):
        hdr[off:off + 4] = np.array([v], dtype=bo + "f4").tobytes()

    i32(0, n), i32(4, n), i32(8, nzv), i32(12, mode)
    i32(28, n), i32(32, n), i32(36, nzv)
    f32(40, n * voxel), f32(44, n * voxel), f32(48, nzv * voxel)
    i32(64, axes[0]), i32(68, axes[1]), i32(72, axes[2])
    i32(92, ext)
    if stamp:
        hdr[208:212] = b"MAP "
    hdr[212:214] = b"\x11\x11" if big_endian else b"\x44\x44"
    dt = {0: "i1", 1: bo + "i2", 2: bo + "f4", 6: bo + "u2", 3: bo + "i2"}[mode]
    payload = np.ascontiguousarray(vol).astype(dt).tobytes()
    if truncate:
        payload = payload[:-truncate]
    with open(path, "wb") as f:
        f.write(bytes(hdr) + b"\0" * ext + payload)


def read_mrc(path):
    raw = open(path, "rb").read()
    n, _, nz, mode = np.frombuffer(raw[:16], dtype="<i4")
    assert mode == 2
    return np.frombuffer(raw[1024:], dtype="<f4").reshape(nz, n, n)
