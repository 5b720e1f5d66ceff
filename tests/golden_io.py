"""Readers for the golden fixtures in tests/golden (written by the reference
itself through oracle/_ref/ref_tool; see tests/golden/make_golden.sh)."""
from __future__ import annotations

import glob
import json
import os
import struct

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def case_dir(name: str) -> str:
    return os.path.join(GOLDEN, name)


def cases(with_ref: str | None = None) -> list[str]:
    out = []
    for d in sorted(glob.glob(os.path.join(GOLDEN, "*", "meta.json"))):
        name = os.path.basename(os.path.dirname(d))
        if with_ref and not os.path.exists(os.path.join(GOLDEN, name, f"ref_{with_ref}.bin")):
            continue
        out.append(name)
    return out


def meta(name: str) -> dict:
    with open(os.path.join(GOLDEN, name, "meta.json")) as f:
        return json.load(f)


def plan_path(name: str, precision: str) -> str:
    return os.path.join(GOLDEN, name, f"plan_{precision}.stnplan")


def read_ref(name: str, precision: str):
    """-> (assignments, values[n, out], scheme_sum or None, (step_count, mults, peak), info json)"""
    path = os.path.join(GOLDEN, name, f"ref_{precision}.bin")
    b = open(path, "rb").read()
    o = 0
    n, oe = struct.unpack_from("<QQ", b, o)
    o += 16
    asg = np.frombuffer(b, np.uint64, n, o).astype(np.int64)
    o += 8 * n
    vals = np.frombuffer(b, np.complex128, n * oe, o).reshape(n, oe)
    o += 16 * n * oe
    (has_sum,) = struct.unpack_from("<Q", b, o)
    o += 8
    s = None
    if has_sum:
        s = np.frombuffer(b, np.complex128, oe, o)
        o += 16 * oe
    bk = struct.unpack_from("<QQQ", b, o)
    with open(os.path.join(GOLDEN, name, f"ref_{precision}.json")) as f:
        info = json.load(f)
    return asg, vals, s, bk, info


def bits(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x).view(np.uint64)
