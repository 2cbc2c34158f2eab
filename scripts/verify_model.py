"""One-off parity check of a whole model on the GPU against the C oracle.

python scripts/verify_model.py resnet20 8   -> sha256 of the GPU's and the
oracle's garbled circuit (reference wire format), decoding tables, garbled
outputs and decoded values for one inference (seed 0x5EED0000, input rng 4000).
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from paper_2302_06361_b200 import models  # noqa: E402
from paper_2302_06361_b200.engine import Dash  # noqa: E402
from pyoracle import Oracle  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
c = models.build(name, 2001, k)
seed = int(0x5EED0000).to_bytes(16, "big")
x = np.random.default_rng(4000).integers(-7, 8, size=(1, c.n_in))
eng = Dash(0)
g = eng.circuit(c)
t = time.time()
net = eng.garble(g, seed)
bo = eng.evaluate(net, eng.garble_inputs(net, x))
out = eng.decode_outputs(net, bo)
gpu = {"gc": hashlib.sha256(net.export_gc(0)).hexdigest(), "dec": hashlib.sha256(net.export_decoding(0)).hexdigest(),
       "gout": hashlib.sha256(bo.payload(0)).hexdigest(), "decoded": out[0].tolist()}
t_gpu = time.time() - t
o = Oracle()
t = time.time()
onet = o.garble(c, seed)
ob = o.evaluate(onet, o.garble_inputs(onet, x[0]))
orc = {"gc": hashlib.sha256(onet.gc_bytes()).hexdigest(), "dec": hashlib.sha256(onet.dec_bytes()).hexdigest(),
       "gout": hashlib.sha256(ob.payload()).hexdigest(), "decoded": o.decode(onet, ob).tolist()}
t_orc = time.time() - t
print(f"{name} k={k}: cts {g.info.cts}  gpu {t_gpu:.1f}s  oracle {t_orc:.1f}s ({os.cpu_count()} threads)")
for key in gpu:
    print(f"  {key:8s} {'MATCH' if gpu[key] == orc[key] else 'DIFF'}  gpu {str(gpu[key])[:64]}  oracle {str(orc[key])[:64]}")
sys.exit(0 if gpu == orc else 1)
