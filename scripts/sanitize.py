"""Small workload for compute-sanitizer (default: Model A batch 1 -- level-
parallel garbling, warp-per-label PRF, lane-group evaluation -- and
model_tiny batch 3; args name:batch), checked against the plain forward pass."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_06361_b200.engine import Dash  # noqa: E402
E = Dash(0)
for name, B in [(a, int(b)) for a, b in (t.split(":") for t in (sys.argv[1:] or ["model_a:1", "model_tiny:3"]))]:
    g = E.model(name, 0 if name == "dense1024" else 1000, 8)
    seeds = b"".join(int(0x5A00 + b).to_bytes(16, "big") for b in range(B))
    x = np.stack([g.random_input(10 + b, -3, 3) for b in range(B)])
    out, _ = E.infer(g, seeds, x)
    try:
        want = [g.plain_forward(xi).tolist() for xi in x]
    except Exception:  # the plain pass overflows the base for some inputs (the GC does not care)
        want = None
    assert want is None or out.tolist() == want, name
print("sanitize workload ok")
