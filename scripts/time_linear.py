"""Times the tensor-core linear kernel alone (garbler pass of one
Dense(1024 -> 1024) layer over B inferences, layer-level API, no decode),
for builds whose results are deliberately wrong (DASH_TC_DBG timing
experiments): python scripts/time_linear.py [B] [lib.so ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_06361_b200.engine import Dash  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
for lib in sys.argv[2:] or [None]:
    E = Dash(0, lib_path=os.path.abspath(lib) if lib else None)
    g = E.model("dense1024", 0, 8)
    seeds = b"".join(int(0x5EED0000 + b).to_bytes(16, "big") for b in range(B))
    net = E.network_setup(g, seeds)
    inp = E.input_base(net)
    E.layer_garble(net, 0, inp)  # warm-up
    E.profile(True)
    for _ in range(3):
        E.layer_garble(net, 0, inp)
    p = E.profile_read()
    E.profile(False)
    ms = p["linear"][0] / 3
    ops = 2 * B * g.info.linear_macs  # one pass, 2 ops per digit-MAC
    print(f"{os.path.basename(lib or 'in-tree')}: B={B} linear {ms:.3f} ms/pass  {ops / ms / 1e9:.3g} int8 ops/s", flush=True)
    del net, inp, E
