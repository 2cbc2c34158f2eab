"""Wall time of the digest parity mode against whole garbling (ResNet-20 k=8)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2302_06361_b200.engine import Dash  # noqa: E402

eng = Dash(0)
g = eng.model("resnet20", 2001, 8)
for B in (1, 16):
    seeds = b"".join((0x5EED0000 + b).to_bytes(16, "big") for b in range(B))
    for name, fn in (("garble", lambda: eng.garble(g, seeds)), ("digest", lambda: eng.garble_digest(g, seeds))):
        r = fn()
        del r
        t = time.perf_counter()
        r = fn()
        print(B, name, round(time.perf_counter() - t, 3), flush=True)
        del r
