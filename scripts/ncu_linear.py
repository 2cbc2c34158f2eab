"""Short workload for ncu captures of the tensor-core linear lanes: one
Dense(1024 -> 1024) garble + eval pass over B inferences (BASELINE
configs[4] linear sweep), or the bench model (lenet5)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_06361_b200.engine import Dash  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
model = sys.argv[2] if len(sys.argv) > 2 else "dense1024"
k = int(sys.argv[3]) if len(sys.argv) > 3 else 8
E = Dash(0)
g = E.model(model, 0 if model == "dense1024" else 2001, k)
seeds = b"".join(int(0x5EED0000 + b).to_bytes(16, "big") for b in range(B))
x = np.random.default_rng(1).integers(-7, 8, size=(B, g.info.n_in)).astype(np.int64)
out, t = E.infer(g, seeds, x)
print("ok", out[0][:4], t.ms_total)
