#!/usr/bin/env python3
"""Golden vectors for the BENCHMARKED batch shapes (tests/golden/golden_batch.json).

Generated from the UNMODIFIED reference (oracle/_ref/libdashref.so, built by
`make -C oracle ref` from /root/reference/proj/core/src) -- or, for circuits
with this repo's Pad2d/Add extensions that the reference cannot run
(ResNet-20), from the C restatement oracle/dash_oracle.c, which is itself
pinned to the reference by tests/test_oracle.py.  Circuits come from the
product's host-only builders (same mt19937 draws as test_models.hpp; equality
with the reference builders is asserted by gen_golden.py).

Records (each inference b: garbling seed, inputs, sha256 of the reference's
wire formats: GC (garble.cpp:347-370), decoding info, garbled inputs,
garbled outputs (bundle_payload, garble.cpp:465-472), decoded values):
  lenet5_b64   BASELINE configs[1] step 0 exactly as bench.py runs it:
               seeds 0x5EED0000 + b, b < 64 (shard.step_seeds(0, 64)),
               inputs numpy default_rng(4000 + b) U[-7, 7]
  minionn_b2   BASELINE configs[2] (paper Model F, k = 9), b < 2
  resnet20_b1  BASELINE configs[3] (k = 8), b < 1, C-oracle generated

usage: python tests/golden/gen_golden_batch.py [lenet5_b64 minionn_b2 resnet20_b1]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from pyoracle import Oracle, RefLib, seed_hex  # noqa: E402

from paper_2302_06361_b200 import models  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_batch.json")

PLAN = {
    # name: (model, builder seed, k, batch, first garbling seed, checker)
    "lenet5_b64": ("lenet5", 2001, 8, 64, 0x5EED0000, "reference"),
    "minionn_b2": ("minionn", 2001, 9, 2, 0x5EED0000, "reference"),
    "resnet20_b1": ("resnet20", 2001, 8, 1, 0x5EED0000, "oracle"),
}


def h(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def batch_inputs(n_in: int, batch: int) -> np.ndarray:
    return np.stack([np.random.default_rng(4000 + b).integers(-7, 8, size=n_in).astype(np.int64)
                     for b in range(batch)])


def record(key):
    model, mseed, k, batch, s0, kind = PLAN[key]
    c = models.build(model, mseed, k)
    lib = RefLib() if kind == "reference" else Oracle()
    ch = lib.circuit(c)
    x = batch_inputs(c.n_in, batch)
    rec = {"model": model, "builder_seed": mseed, "k": k, "batch": batch, "first_seed": hex(s0),
           "inputs": "numpy default_rng(4000 + b).integers(-7, 8, n_in)", "checker": kind, "inferences": []}
    t0 = time.time()
    for b in range(batch):
        net = lib.garble(ch, seed_hex(s0 + b))
        gc = net.gc_bytes()
        bi = lib.garble_inputs(net, x[b])
        bo = lib.evaluate(net, bi)
        dec = lib.decode(net, bo)
        rec["inferences"].append({"b": b, "gc": h(gc), "gc_len": len(gc), "dec": h(net.dec_bytes()),
                                  "gin": h(bi.payload()), "gout": h(bo.payload()), "decoded": dec.tolist()})
        del gc, net
        print(f"{key} b={b} {time.time() - t0:.1f}s", flush=True)
    return rec


def main():
    keys = sys.argv[1:] or list(PLAN)
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    out["generator"] = "tests/golden/gen_golden_batch.py (reference: oracle/_ref/libdashref.so; " \
                       "extensions: oracle/liboracle.so)"
    for k in keys:
        out[k] = record(k)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
