"""The reference's binary dense-matrix format (io.hpp:8-17, io.cpp:44-72):
16-byte little-endian header (magic u32 0x54414D44 "DMAT", rows u64, cols
u32) followed by rows*cols binary64 values in row-major order. Used to feed
identical bytes to the CPU oracle and the device."""
import struct

import numpy as np

MAGIC = 0x54414D44


def save_dmat(path, a):
    a = np.ascontiguousarray(a, dtype="<f8")
    if a.ndim != 2:
        raise ValueError("save_dmat: expected a matrix")
    with open(path, "wb") as f:
        f.write(struct.pack("<IQI", MAGIC, a.shape[0], a.shape[1]))
        f.write(a.tobytes())


def load_dmat(path):
    with open(path, "rb") as f:
        head = f.read(16)
        if len(head) != 16:
            raise ValueError(f"not a .dmat file: {path}")
        magic, rows, cols = struct.unpack("<IQI", head)
        if magic != MAGIC:
            raise ValueError(f"not a .dmat file: {path}")
        data = np.frombuffer(f.read(), dtype="<f8")
    if data.size != rows * cols:
        raise ValueError(f"truncated .dmat file: {path}")
    return data.reshape(rows, cols).astype(np.float64)
