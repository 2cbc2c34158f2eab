"""compute-sanitizer workload for the streamed-garbling paths (DESIGN.md
§11.1): layer-windowed dashgpu_infer, dashgpu_garble_digest and
dashgpu_garble_stream on model_tiny (private weights) and Model F dims
(residual DAG, empty layers), checked against the whole-GC schedule."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_06361_b200.engine import Dash  # noqa: E402

E = Dash(0)
for name, seed, k, priv in [("model_tiny", 1000, 8, True), ("model_f_dims", 1006, 9, False)]:
    g = E.model(name, seed, k, priv)
    B = 2
    seeds = b"".join(int(0x5B00 + b).to_bytes(16, "big") for b in range(B))
    x = np.stack([g.random_input(20 + b, -3, 3) for b in range(B)])
    os.environ["DASHGPU_LAYERWISE"] = "1"
    lw, t = E.infer(g, seeds, x)
    os.environ["DASHGPU_LAYERWISE"] = "0"
    whole, _ = E.infer(g, seeds, x)
    assert t.layerwise == 1 and (lw == whole).all(), name
    dg = E.garble_digest(g, seeds)
    h = {}
    E.garble_stream(g, seeds, lambda b, d: h.setdefault(b, hashlib.sha256()).update(d))
    net = E.garble(g, seeds)
    for b in range(B):
        assert h[b].digest() == hashlib.sha256(net.export_gc(b)).digest(), name
    assert dg.shape == (B, g.info.n_layers, 32)
    for b in range(B):
        assert (net.digest(b) == dg[b]).all(), name
        assert (E.import_gc([net.export_gc(b)], host_resident=True).digest(0) == dg[b]).all(), name
print("sanitize stream workload ok")
