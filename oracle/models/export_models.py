#!/usr/bin/env python3
"""Writes the benchmark circuits as plain weight files (oracle/models/*.npz).

TEST / BASELINE INFRASTRUCTURE.  bench.py's reference arm (--impl reference)
and cpu_baseline leg load these files and hand them to the unmodified
reference (oracle/_ref) or the C restatement, so the CPU baseline process
never loads the product library.  The weights were drawn by the product's
host-only builders, which reproduce the reference's mt19937 draws
(tests/support/test_models.hpp; equality asserted by
tests/golden/gen_golden.py for the models the reference itself defines).

usage: python oracle/models/export_models.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from paper_2302_06361_b200 import models  # noqa: E402
from pyoracle import save_circuit  # noqa: E402

PLAN = [("lenet5", 2001, 8), ("minionn", 2001, 9), ("resnet20", 2001, 8), ("model_a", 2001, 8)]

if __name__ == "__main__":
    for name, seed, k in PLAN:
        path = os.path.join(HERE, f"{name}_s{seed}_k{k}.npz")
        save_circuit(models.build(name, seed, k), path)
        print("wrote", path, os.path.getsize(path), "bytes")
