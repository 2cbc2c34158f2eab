"""Shared helpers for the parity tests."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2302_06361_b200 import models  # noqa: E402

PRIMES = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53]


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def seed_hex(v: int) -> bytes:
    """seed_from_string(hex(v)) of the reference: big-endian 16 bytes (prf.cpp:42-66)."""
    return int(v).to_bytes(16, "big")


def golden_circuit(rec):
    """Rebuilds the circuit of a golden network record."""
    tag = rec["tag"]
    parts = tag.split("/")
    name = parts[0]
    if "target" in parts[1]:
        tgt = float(parts[1][len("target"):])
        k = int(parts[2][1:])
        seed = 1000 if name == "model_tiny" else 0
        c = models.build(name, seed, k)
        c.sign_target = tgt
        return c
    seed = int(parts[1][1:])
    k = int(parts[2][1:])
    priv = parts[3] == "priv"
    return models.build(name, seed, k, priv)


def golden_input(rec, inp, n_in):
    lo, hi = rec["input_range"]
    return np.random.default_rng(inp["rng"]).integers(lo, hi + 1, size=n_in).astype(np.int64)


def u128_pairs(vals):
    return np.array([[v & ((1 << 64) - 1), v >> 64] for v in vals], dtype=np.uint64)


def pairs_u128(a):
    return [int(x[0]) | (int(x[1]) << 64) for x in a]
