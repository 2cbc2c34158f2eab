"""Development probe: parity spot checks + first timings on the GPU box."""
import hashlib, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import __graft_entry__
from paper_2302_06361_b200.engine import Dash
from pyoracle import Oracle, seed_hex

__graft_entry__.smoke()
E = Dash(0); O = Oracle()
rnd = np.random.default_rng(1)
for m in [2,3,5,7,8,9,11,13,33,46,64,110,127,128]:
    vals = rnd.integers(0, 2**63, size=(256,2), dtype=np.uint64)
    out, dg = E.prim(0, m, inp=vals)
    for i in range(256):
        c = int(vals[i,0]) | (int(vals[i,1])<<64)
        want = O.decompress_mod(c, m)
        assert list(dg[i,:len(want)]) == want, (m, i)
print("codec ok", flush=True)
for name, s, k, sd in [("model_a",1001,8,0xe2e0a1), ("model_c",1003,9,0xc0), ("model_tiny",1000,8,0x77)]:
    g = E.model(name, s, k)
    net = E.garble(g, seed_hex(sd) + seed_hex(sd+1))
    onet = O.garble(g.to_circuit(), seed_hex(sd))
    a = net.export_gc(0); b = onet.gc_bytes()
    print(name, "gc equal:", a == b, hashlib.sha256(a).hexdigest()[:16], flush=True)
    x = np.stack([g.random_input(4000), g.random_input(4001)])
    d = E.decode_outputs(net, E.evaluate(net, E.garble_inputs(net, x)))
    want = O.decode(onet, O.evaluate(onet, O.garble_inputs(onet, x[0])))
    print("  decoded equal:", (d[0] == want).all(), d[0][:4], flush=True)
for name, k, B in [("lenet5", 8, 64), ("model_a", 8, 64)]:
    g = E.model(name, 2001, k)
    print(name, "cts/inf", g.info.cts, "relu elems", g.info.relu_elements, flush=True)
    seeds = b"".join(seed_hex(0x5eed0000 + b) for b in range(B))
    x = np.stack([g.random_input(4000 + b) for b in range(B)])
    for it in range(3):
        E.profile(True)
        t = time.time(); out, tm = E.infer(g, seeds, x); dt = time.time() - t
        prof = E.profile_read()
        print(f"  iter {it}: {dt*1e3:.1f} ms wall -> {B/dt:.1f} inf/s; garble {tm.ms_garble:.1f} eval {tm.ms_evaluate:.1f} encode {tm.ms_encode:.1f} decode {tm.ms_decode:.1f}", flush=True)
        print("   ", {k: (round(v[0], 2), v[1]) for k, v in prof.items() if v[1]}, flush=True)
