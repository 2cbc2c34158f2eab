"""A/B timing of library variants: python scripts/exp_time.py lib1.so lib2.so ..."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_06361_b200.engine import Dash
B = 64
for path in sys.argv[1:]:
    E = Dash(0, lib_path=os.path.abspath(path))
    g = E.model("lenet5", 2001, 8)
    seeds = b"".join(int(0x5EED0000 + b).to_bytes(16, "big") for b in range(B))
    x = np.random.default_rng(1).integers(-7, 8, size=(B, g.info.n_in)).astype(np.int64)
    E.infer(g, seeds, x)
    E.profile(True)
    t = time.time()
    for _ in range(4):
        out, _ = E.infer(g, seeds, x)
    dt = (time.time() - t) / 4
    p = E.profile_read()
    print(f"{os.path.basename(path)}: {B/dt:.1f} inf/s  act_garble {p['act_garble'][0]/4:.2f} ms  act_eval {p['act_eval'][0]/4:.2f} ms  out0={out[0][:3]}", flush=True)
    print("   " + "  ".join(f"{k} {v[0]/4:.2f}ms/{v[1]//4}" for k, v in p.items() if v[1]), flush=True)
    del E
