"""Digest parity mode beyond HBM: garble ResNet-20 k=8 for
B inferences whose GCs together exceed the GPU's memory through the
one-layer window (dashgpu_garble_digest), then garble single inferences
whole and check their per-layer digests (dashgpu_network_digest) against
the streamed ones."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2302_06361_b200.engine import Dash  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 40
eng = Dash(0)
g = eng.model("resnet20", 2001, 8)
seeds = [(0x5EED0000 + b).to_bytes(16, "big") for b in range(B)]
gc_rows = g.info.cts * 16
t = time.perf_counter()
dg = eng.garble_digest(g, b"".join(seeds))
dt = time.perf_counter() - t
checked = []
for b in (0, B // 2, B - 1):
    net = eng.garble(g, seeds[b])
    assert (net.digest(0) == dg[b]).all(), b
    checked.append(b)
    del net
print(json.dumps({"workload": f"resnet20 k=8, {B} inferences", "gc_row_bytes_total": gc_rows * B,
                  "gc_row_GB_per_inference": gc_rows / 1e9, "digest_s": dt,
                  "inferences_per_s": B / dt, "row_GB_per_s": gc_rows * B / dt / 1e9,
                  "checked_whole_gc_digests": checked}))
