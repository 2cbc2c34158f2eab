"""Evaluation from a host-resident GC (dashgpu_import_gc_host: rows in pinned
host memory, moved to a one-layer device window per layer) against an HBM
import, LeNet-5 k=8.  Wall clock around evaluate (which
returns after its stream work)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2302_06361_b200.engine import Dash  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
eng = Dash(0)
g = eng.model("lenet5", 2001, 8)
net = eng.garble(g, b"".join((0x5EED0000 + b).to_bytes(16, "big") for b in range(B)))
x = np.stack([g.random_input(4000 + b) for b in range(B)])
bi = eng.garble_inputs(net, x)
gcs = [net.export_gc(b) for b in range(B)]
payload = b"".join(bi.payload(b) for b in range(B))
res = {"workload": f"lenet5 k=8 batch {B}", "gc_bytes": sum(len(c) for c in gcs)}
outs = {}
for mode in ("hbm", "host"):
    ev = eng.import_gc(gcs, host_resident=(mode == "host"))
    inb = eng.import_bundle(ev, payload, False)
    eng.evaluate(ev, inb)  # warm-up
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        o = eng.evaluate(ev, inb)
        o.payload(0)
        best = min(best, time.perf_counter() - t)
    outs[mode] = [o.payload(b) for b in range(B)]
    res[f"{mode}_evaluate_s"] = best
    res[f"{mode}_inferences_per_s"] = B / best
    res[f"{mode}_GC_GBps"] = res["gc_bytes"] / best / 1e9
    del ev, inb, o
assert outs["hbm"] == outs["host"]
print(json.dumps(res))
