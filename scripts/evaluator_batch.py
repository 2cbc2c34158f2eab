"""Evaluator service throughput (best of three runs per mode): N sessions of one circuit answered one by one
(EvaluatorService.handle, one device network per session) vs as a batch
(handle_batch: one dashgpu_import_gc of N GCs, one evaluation launch).
Prints one JSON line; wall-clock around the calls (each returns after a sync)."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_06361_b200.engine import Dash
from paper_2302_06361_b200 import protocol as P

model = sys.argv[1] if len(sys.argv) > 1 else "lenet5"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 32
eng = Dash(0)
g = eng.model(model, 2001, 8)
seeds = b"".join(int(0xE0A0 + i).to_bytes(16, "big") for i in range(N))
net = eng.garble(g, seeds)
x = np.random.default_rng(3).integers(-7, 8, size=(N, g.info.n_in)).astype(np.int64)
bi = eng.garble_inputs(net, x)
gcs = [net.export_gc(i) for i in range(N)]
gins = [bi.payload(i) for i in range(N)]
T = P.FrameType


def run(batched, base):
    ev = P.EvaluatorService(eng)
    t0 = time.perf_counter()
    if batched:
        ev.handle_batch([P.Frame(T.GC_TRANSFER, base + i, gcs[i]) for i in range(N)])
    else:
        for i in range(N):
            ev.handle(P.Frame(T.GC_TRANSFER, base + i, gcs[i]))
    t1 = time.perf_counter()
    if batched:
        outs = ev.handle_batch([P.Frame(T.GARBLED_INPUT, base + i, gins[i]) for i in range(N)])
    else:
        outs = [ev.handle(P.Frame(T.GARBLED_INPUT, base + i, gins[i])) for i in range(N)]
    t2 = time.perf_counter()
    pay = {f.session - base: f.payload for f in outs}
    return t1 - t0, t2 - t1, pay


run(False, 1 << 20)  # warm-up (allocations, module load)
run(True, 2 << 20)
# best of three fresh service instances per mode (sessions are single-use)
r1 = [run(False, (3 + k) << 20) for k in range(3)]
rb = [run(True, (6 + k) << 20) for k in range(3)]
imp1, ev1, p1 = min(r1, key=lambda r: r[1])
impb, evb, pb = min(rb, key=lambda r: r[1])
imp1, impb = min(r[0] for r in r1), min(r[0] for r in rb)
assert p1 == pb and len(pb) == N
print(json.dumps({"model": model, "sessions": N, "gc_mb_per_session": len(gcs[0]) / 1e6,
                  "one_by_one": {"gc_import_s": imp1, "online_eval_s": ev1, "sessions_per_s_online": N / ev1},
                  "batched": {"gc_import_s": impb, "online_eval_s": evb, "sessions_per_s_online": N / evb},
                  "online_speedup": ev1 / evb, "payloads_identical": True}))
