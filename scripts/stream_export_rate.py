"""GC bytes/s of the streamed export (dashgpu_garble_stream) against garble +
export_gc per inference, LeNet-5 k=8.  Wall clock around
the calls: both include the host copies, which is what a garbler pays."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2302_06361_b200.engine import Dash  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
eng = Dash(0)
g = eng.model("lenet5", 2001, 8)
seeds = b"".join((0x5EED0000 + b).to_bytes(16, "big") for b in range(B))
total = [0]


def sink(b, data):
    total[0] += len(data)


eng.garble_stream(g, seeds[:16], sink)  # warm-up
total[0] = 0
t = time.perf_counter()
eng.garble_stream(g, seeds, sink)
ts = time.perf_counter() - t
nbytes = total[0]
t = time.perf_counter()
net = eng.garble(g, seeds)
for b in range(B):
    net.export_gc(b)
tw = time.perf_counter() - t
print(json.dumps({"workload": f"lenet5 k=8 batch {B}", "gc_bytes": nbytes,
                  "streamed_s": ts, "streamed_GBps": nbytes / ts / 1e9,
                  "whole_then_export_s": tw, "whole_then_export_GBps": nbytes / tw / 1e9}))
