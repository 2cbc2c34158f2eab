#!/usr/bin/env python3
"""Measured int8 tensor-core peak of this B200 (the linear lanes' roofline
denominator): cuBLASLt int8 GEMM (torch._int_mm, s8 x s8
-> s32) at 8192^3 and a few other square / skinny shapes, CUDA events, best
of the timed repetitions.  A yardstick only: the product's linear lanes are
the hand-written tcgen05 kernel.  Writes profiles/int8_peak.json.

    python scripts/int8_peak.py [--out profiles/int8_peak.json]
"""
import argparse
import json
import os
import subprocess

import torch


def clocks():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,name", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=10).stdout.strip()
        return out
    except Exception:
        return None


def bench(M, N, K, reps=20):
    a = torch.randint(-128, 127, (M, K), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (K, N), dtype=torch.int8, device="cuda").t().contiguous().t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return 2.0 * M * N * K / best / 1e12, best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "profiles", "int8_peak.json"))
    args = ap.parse_args()
    shapes = [(8192, 8192, 8192), (16384, 16384, 8192), (4096, 4096, 4096), (16384, 1024, 1024)]
    res = []
    for M, N, K in shapes:
        tops, sec = bench(M, N, K)
        res.append({"M": M, "N": N, "K": K, "tops": tops, "seconds": sec})
        print(json.dumps(res[-1]), flush=True)
    best = max(r["tops"] for r in res)
    out = {"tops": best, "unit": "TOPS (int8 dense, 2 ops per MAC)",
           "how": "cuBLASLt int8 GEMM via torch._int_mm, best over shapes (scripts/int8_peak.py)",
           "shapes": res, "clocks": clocks(), "device": torch.cuda.get_device_name(0)}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({"int8_peak_tops": best}))


if __name__ == "__main__":
    main()
