"""CPU baselines of the large configs on the GPU box's host cores (bounded
samples, as bench.py's cpu_baseline leg): python scripts/cpu_baselines.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

for model, k, sample in (("minionn", 9, 4), ("resnet20", 8, 2), ("model_a", 8, 64)):
    bench.MODEL_NAME[0] = model
    c = bench.reference_circuit(model, k)
    r = bench.cpu_baseline(c, c.n_in, c.n_out, sample)
    r["model"], r["k"] = model, k
    print(json.dumps(r), flush=True)
