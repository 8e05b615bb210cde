"""Shared helpers for the GPU parity tests: seeded inputs exactly as the
reference's random_inputs produces them (restated in oracle/oracle.c and
pinned to the reference in tests/test_oracle.py), and torch/numpy plumbing."""
from __future__ import annotations

import numpy as np
import torch

from oracle.pyoracle import Orc


def conv_inputs(n, hp, wp, c, k, r, s, seed, fp16=False, with_seed=True):
    """random_inputs of conv2d_nhwc_tdsl(...): data=seed+0, kernel=seed+1, out=seed+2."""
    d, w, a = ("fp16", "fp16", "fp32") if fp16 else ("u8", "i8", "i32")
    st_oh = None  # computed by caller
    x = Orc.random_tensor(d, (n, hp, wp, c), seed)
    wt = Orc.random_tensor(w, (k, r, s, c), seed + 1)
    return x, wt


def out_seed(shape, seed, fp16=False):
    return Orc.random_tensor("fp32" if fp16 else "i32", shape, seed)


def to_dev(a: np.ndarray, dev, f16=False):
    t = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    if f16:
        t = t.view(torch.float16)
    return t


def rel_dev(ref: np.ndarray, got: np.ndarray) -> float:
    """max |a-b| / max(|ref|, 1) — the reference's compare() (vm.cpp:626-639)."""
    ref = ref.astype(np.float64)
    got = got.astype(np.float64)
    return float(np.max(np.abs(ref - got) / np.maximum(np.abs(ref), 1.0))) if ref.size else 0.0


def read_tnsr(path):
    """numpy view of a TNSR container (proj/src/vm.cpp:686-822 layout)."""
    import struct

    import numpy as np
    raw = open(path, "rb").read()
    assert raw[:4] == b"TNSR" and raw[4] == 1
    dt = [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.float16, np.float32][raw[5]]
    rank = raw[6]
    shape = struct.unpack("<%dQ" % rank, raw[7:7 + 8 * rank])
    return np.frombuffer(raw[7 + 8 * rank:], dtype=dt).reshape(shape)
