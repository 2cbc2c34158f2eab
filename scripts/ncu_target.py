"""Short workload for ncu captures: one garble+eval pass of the bench model."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_06361_b200.engine import Dash
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
model = sys.argv[2] if len(sys.argv) > 2 else "lenet5"
E = Dash(0)
g = E.model(model, 2001, 8)
seeds = b"".join(int(0x5EED0000 + b).to_bytes(16, "big") for b in range(B))
x = np.random.default_rng(1).integers(-7, 8, size=(B, g.info.n_in)).astype(np.int64)
out, t = E.infer(g, seeds, x)
print("ok", out[0][:4], t.ms_total)
