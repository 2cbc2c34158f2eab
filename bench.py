#!/usr/bin/env python3
"""Benchmark: garbled inferences/s (garble + garble_inputs + evaluate + decode).

Workload (BASELINE.json configs[1]): LeNet-5 restated in reference ops on
synthetic 28x28 inputs, batch 64 per GPU, k = 8 CRT primes, one fresh seed per
inference per step (garbled circuits are single-use).  A step garbles,
encodes, evaluates and decodes the whole batch; the per-step garbled tables
(8 GB at batch 64) are far larger than L2, so no explicit flush is needed.

  value   inputs (seeds + quantized inputs) already in HBM, outputs left in HBM,
          CUDA events on the stream the library launches on, max over ranks.
  e2e     the same metric through the C-ABI call dashgpu_infer with HOST
          buffers: H2D of seeds + inputs and D2H of the decoded outputs inside
          the timed region.
  kernels the library's per-launch CUDA events (kernels_ms_per_step, the
          roofline's kernel duration) come from a second, untimed pass of
          the same steps, so their host cost does not enter `value`.
  --impl reference: the reference's own CPU implementation (oracle/_ref, the
          unmodified dash_core sources) on the host cores, rank 0 only.

Multi-GPU (torchrun): inferences are sharded across ranks (weak scaling), the
decoded outputs are all-gathered over NCCL once per step.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODEL, SEED, K = "lenet5", 2001, 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--model", default=MODEL)
    ap.add_argument("--k", type=int, default=K)
    ap.add_argument("--private", action="store_true", help="private-weight linear layers (projection per weight, "
                                                           "the JSON model default, model_io.cpp:56)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="inferences in the CPU-baseline sample")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline (config sweeps)")
    ap.add_argument("--sweep", default="", help="label-ops sweep (BASELINE configs[4]): 'proj' (ReLU layer), "
                                                "'tproj' (raw projection gates) and/or 'linear' (Dense 1024^2), "
                                                "comma separated; --sweep-log2 / --sweep-k select the grid")
    ap.add_argument("--sweep-log2", default="16,18,20,22,24,26")
    ap.add_argument("--sweep-k", default="2,4,6,8")
    ap.add_argument("--emulate", action="store_true", help=argparse.SUPPRESS)  # tests: CPU emulation + gloo
    return ap.parse_args()


def seeds_for(step, rank, world, batch):
    """This rank's shard of the step's fresh seeds (paper_2302_06361_b200.shard)."""
    from paper_2302_06361_b200.shard import shard_range, step_seeds

    a, b = shard_range(world * batch, world, rank)
    return b"".join(step_seeds(step, world * batch)[a:b])


class ClockSampler:
    """SM clocks and throttle reasons during the timed region.

    NVML (pynvml) is polled every 2 ms from a thread for the first 250
    samples, so even a timed region of a few milliseconds (Model A batch 1)
    gets samples, and every 20 ms after that; nvidia-smi -lms 100
    is the fallback when NVML is unavailable."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, {reason names})
        self.proc = None
        self.nvml = None
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            self.nvml = (N, N.nvmlDeviceGetHandleByIndex(idx))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        N, h = self.nvml
        bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            N.nvmlDeviceGetCurrentClocksThrottleReasons
        while True:
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = reasons(h)
                self.rows.append((float(sm), float(mx), {n for n, b in bits.items() if r & b}))
            except Exception:
                pass
            # 2 ms for the first ~0.5 s (short regions get samples), then 20 ms:
            # NVML queries take driver locks the CUDA host calls also need
            if self._stop.wait(0.002 if len(self.rows) < 250 else 0.02):
                return

    def _read(self):
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            try:
                self.rows.append((float(r[0]), float(r[1]),
                                  {self.NAMES[i] for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"}))
            except (ValueError, IndexError):
                pass

    def __exit__(self, *a):
        self._stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.t is not None:
            self.t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(set().union(*(r[2] for r in self.rows))), "samples": len(self.rows),
                "sampler": "nvml 2 ms x 250, then 20 ms" if self.nvml else "nvidia-smi 100 ms"}


def cpu_baseline(circuit_desc_c, n_in, n_out, sample):
    """Reference CPU path (oracle/_ref) on the host cores, bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle

    cores = os.cpu_count() or 1
    ref_ok = pyoracle.have_ref()
    if ref_ok:
        try:
            R = pyoracle.RefLib()
            ch = R.circuit(circuit_desc_c)
        except Exception:  # circuits with this repo's extensions (ResNet-20): the reference cannot run them
            ref_ok = False
    if ref_ok:
        kind = "reference"
        seeds = b"".join(int(0x5EED0000 + b).to_bytes(16, "big") for b in range(sample))
        rng = np.random.default_rng(7)
        x = rng.integers(-7, 8, size=(sample, n_in)).astype(np.int64)
        best = None
        # inference-parallel (one inference per core) when the sample fills the
        # cores, and the reference's intra-layer OpenMP mode
        for mode in ((1, 0) if sample >= cores else (0,)):
            sec, _ = R.bench_infer(ch, seeds, x, mode, cores)
            v = sample / sec
            if best is None or v > best[0]:
                best = (v, mode, sec)
        return {"value": best[0], "unit": "inferences/s", "cores": cores, "kind": kind, "cpu": host_cpu(),
                "sample": f"{sample} {MODEL_NAME[0]} inferences (garble+garble_inputs+evaluate+decode_outputs), "
                          f"{'inference-parallel' if best[1] == 1 else 'OpenMP intra-layer'} on {cores} threads, "
                          f"{best[2]:.1f} s"}
    O = pyoracle.Oracle()
    ch = O.circuit(circuit_desc_c)
    seeds = b"".join(int(0x5EED0000 + b).to_bytes(16, "big") for b in range(sample))
    x = np.random.default_rng(7).integers(-7, 8, size=(sample, n_in)).astype(np.int64)
    sec, _ = O.bench_infer(ch, seeds, x, cores)
    mode = "inference-parallel" if sample >= cores else "OpenMP intra-layer"
    return {"value": sample / sec, "unit": "inferences/s", "cores": cores, "kind": "port", "cpu": host_cpu(),
            "sample": f"{sample} {MODEL_NAME[0]} inferences, C oracle port (the reference has no Pad2d/Add layers), "
                      f"{mode} on {cores} threads, {sec:.1f} s"}


MODEL_NAME = [MODEL]
WORKLOADS = {
    "lenet5": "LeNet-5 restated in reference ops, 1x28x28",
    "model_a": "784-128-128-10 ReLU MLP, testsupport::model_a",
    "minionn": "paper Model F, MiniONN-style 7-conv CIFAR CNN, 3x32x32, ReLU",
    "resnet20": "ResNet-20 CIFAR, 3x32x32, Pad2d/Add/DAG extensions, ReLU",
    "resnet20s": "ResNet-20 CIFAR, SignAct after every residual add",
    "model_c": "testsupport::model_c", "model_d": "testsupport::model_d",
}


def host_cpu():
    """lscpu-style model string of the host (state the CPU)."""
    name, fam, model = "unknown", "?", "?"
    try:
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name":
                name = v
            elif k == "cpu family":
                fam = v
            elif k == "model":
                model = v
            if name != "unknown" and fam != "?" and model != "?":
                break
    except OSError:
        pass
    return f"{name} (family {fam} model {model}), {os.cpu_count()} logical CPUs"


def reference_circuit(model, k):
    """The benchmark circuit as a plain weight file (oracle/models/*.npz,
    written by oracle/models/export_models.py): the reference arm hands it to
    the unmodified reference without loading the product library."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle

    path = os.path.join(ROOT, "oracle", "models", f"{model}_s{SEED}_k{k}.npz")
    if not os.path.exists(path):
        raise SystemExit(f"no weight file {path}; run oracle/models/export_models.py")
    return pyoracle.load_circuit(path)


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation, rank 0 only.

    Same workload as the GPU arm: each timed step garbles, encodes, evaluates
    and decodes args.batch fresh inferences (64 for the headline) on the
    unmodified reference (oracle/_ref: proj/core/src/*.cpp, -O2
    -march=native) with one inference per core (inference-parallel; the
    reference has no batching, so this is its best mode for a batch).  The
    untimed warm-up steps run one inference per core."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle

    c = reference_circuit(args.model, args.k)
    for l in c.layers:  # --private: projection per weight (model_io.cpp:56 default)
        l.private_weights = bool(args.private and l.linear())
    cores = os.cpu_count() or 1
    n_in = c.n_in
    if pyoracle.have_ref():
        try:
            R = pyoracle.RefLib()
            ch = R.circuit(c)
            kind = "reference"
        except pyoracle.CheckerError:  # Pad2d / Add extensions (ResNet-20): the reference cannot run them
            R = None
    else:
        R = None
    if R is None:
        O = pyoracle.Oracle()
        ch = O.circuit(c)
        kind = "port"

    def step(i, n):
        seeds = b"".join(int(0x5EED0000 + i * n + b).to_bytes(16, "big") for b in range(n))
        x = np.random.default_rng(i).integers(-7, 8, size=(n, n_in)).astype(np.int64)
        if R is not None:
            return R.bench_infer(ch, seeds, x, 1, cores)[0]
        return O.bench_infer(ch, seeds, x, cores)[0]

    for i in range(args.warmup):
        step(i, min(args.batch, cores))
    total = 0.0
    for i in range(args.steps):
        total += step(args.warmup + i, args.batch)
    value = args.batch * args.steps / total
    line = {"metric": "garbled inferences/sec (garble+eval)", "value": value, "unit": "inferences/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"{args.model}{' (private weights)' if args.private else ''} "
                                   f"({WORKLOADS.get(args.model, 'single-layer sweep')}) k={args.k}, "
                                   f"synthetic inputs U[-7,7], batch {args.batch} per step, fresh seed per "
                                   f"inference per step",
                       "global_batch": args.batch, "inferences_per_gpu": args.batch,
                       "parallelism": f"reference CPU path, inference-parallel on {cores} cores"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "inferences/s", "cores": cores, "kind": kind,
                             "cpu": host_cpu(),
                             "sample": f"{args.batch} inferences per step x {args.steps} timed steps "
                                       f"(garble+garble_inputs+evaluate+decode_outputs, one inference per core); "
                                       f"warm-up steps {min(args.batch, cores)} inferences",
                             "build": "oracle/_ref: unmodified proj/core/src/*.cpp, g++ -O2 -march=native -fopenmp"
                             if kind == "reference" else "oracle/liboracle.so (C restatement)"},
            "e2e": {"value": value, "unit": "inferences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_sweep(args):
    """Label-ops sweep (BASELINE configs[4]).

    proj:   one ReLU layer of N = 2^j elements ({input_shape={N}, layers={relu()}},
            reference bench_main.cpp:156-162), garbled + evaluated + decoded in
            element chunks through dashgpu_infer_stream; a projection label-op is
            one garbled row (garble) or one decrypted row (eval).
    linear: Dense(1024 -> 1024) over B = N / 1024 inferences through
            dashgpu_infer; a linear label-op is one label x scalar MAC (n_p digit
            MACs), timed on the tcgen05 linear kernel's CUDA events.
    One JSON line per grid point, all on one GPU (the sweep shards by element
    range / CRT lane with no exchange)."""
    import torch
    import torch.distributed as dist
    from paper_2302_06361_b200.engine import Dash
    from paper_2302_06361_b200.shard import shard_range

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:  # proj: element-range shards of the layer; linear: inference shards
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def max_over_ranks(sec):
        if world == 1:
            return sec
        t = torch.tensor([sec], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    eng = Dash(local)
    eng.set_stream(torch.cuda.current_stream().cuda_stream)
    kinds = [s for s in args.sweep.split(",") if s]
    PR = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53]

    def timed(fn):
        """fn() between CUDA events on the library's stream (torch's current
        stream), max over ranks; returns (device seconds, wall seconds)."""
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        return max_over_ranks(e0.elapsed_time(e1) / 1e3), max_over_ranks(wall), r

    for kind in kinds:
        for j in [int(v) for v in args.sweep_log2.split(",")]:
            for k in [int(v) for v in args.sweep_k.split(",")]:
                N = 1 << j
                if kind == "proj":
                    g = eng.model(f"relu{N}", 0, k)
                    info = g.info
                    P = 1
                    for p in PR[:k]:
                        P *= p
                    x = np.random.default_rng(j * 16 + k).integers(-(P // 2), (P + 1) // 2, size=(1, N))
                    chunk = min(N, max(1 << 14, int(24e9 // (16 * info.act_uc_cts))))
                    a, b = shard_range(N, world, rank)
                    chunk = min(chunk, max(1, b - a))
                    # warm-up on the same circuit at the timed chunk size: the
                    # stream workspace is allocated here and reused by the timed call
                    eng.infer_stream(g, (0x5EED).to_bytes(16, "big"), x, chunk, u_range=(a, a + chunk))
                    sec, wall, (out, tm, _) = timed(lambda: eng.infer_stream(
                        g, (0x5EED0001).to_bytes(16, "big"), x, chunk, u_range=(a, b)))
                    assert (out[0, a:b] == np.maximum(x[0, a:b], 0)).all(), "ReLU sweep mismatch"
                    rows = N * (info.act_uc_cts + info.act_eval_rows)
                    line = {"sweep": "proj", "labels": N, "k": k, "n_gpus": world, "label_ops_per_s": rows / sec,
                            "elements_per_s": N / sec, "seconds": sec, "wall_seconds": wall,
                            "garbled_rows": N * info.act_uc_cts, "eval_rows": N * info.act_eval_rows,
                            "table_bytes": 16 * N * info.act_uc_cts,
                            "table_GBps": 16 * N * info.act_uc_cts / sec / 1e9, "chunk_elements": chunk,
                            "chunks": tm.sub_batches, "check": "decoded == ReLU(x) for every element",
                            "roofline": {"bound": "hbm", "achieved": 16 * N * info.act_uc_cts / sec / 1e9,
                                         "peak": measured_peaks()[0], "unit": "GB/s",
                                         "frac": 16 * N * info.act_uc_cts / sec / 1e9 / measured_peaks()[0],
                                         "note": "garbled-table bytes over the whole streamed layer; the gadget "
                                                 "tape is integer-issue bound (AES + label codec)"},
                            "workload": "{input_shape={N}, layers={relu()}} (bench_main.cpp:156-162), garble + "
                                        "garble_inputs + evaluate + decode, streamed in element chunks"}
                elif kind == "tproj":
                    # raw t_proj (bench_main.cpp:40-74, phi(a) = a^2 + 1 mod p): N gates per CRT lane,
                    # garbled (p rows each) then evaluated (one row each), device-resident
                    a, b = shard_range(N, world, rank)
                    n = max(1, b - a)
                    pmax = max(PR[:k])
                    gen = torch.Generator(device="cuda").manual_seed(j * 16 + k)
                    lab = torch.randint(-2**62, 2**62, (n, 2), dtype=torch.int64, device="cuda", generator=gen)
                    gates = torch.arange(a, a + n, dtype=torch.int64, device="cuda")
                    wires = gates + N
                    rows = torch.empty((n * pmax, 2), dtype=torch.int64, device="cuda")
                    out0 = torch.empty((n, 2), dtype=torch.int64, device="cuda")
                    outv = torch.empty((n, 2), dtype=torch.int64, device="cuda")
                    seed = (0x7B0 + k).to_bytes(16, "big")
                    ctxs = [eng.proj_ctx(seed, p, p, [(v * v + 1) % p for v in range(p)]) for p in PR[:k]]
                    for c in ctxs:  # warm-up
                        c.garble(min(n, 4096), lab.data_ptr(), gates.data_ptr(), wires.data_ptr(),
                                 rows.data_ptr(), out0.data_ptr())
                    tg = te = 0.0
                    for c in ctxs:
                        dg, _, _ = timed(lambda: c.garble(n, lab.data_ptr(), gates.data_ptr(), wires.data_ptr(),
                                                          rows.data_ptr(), out0.data_ptr()))
                        # evaluate on the base labels (= the active labels of value 0: colour-random rows)
                        de, _, _ = timed(lambda: c.eval(n, lab.data_ptr(), gates.data_ptr(), rows.data_ptr(),
                                                        outv.data_ptr()))
                        tg, te = tg + dg, te + de
                        # property check on a sample: eval(x0) == out0 + phi(0) R_q = out0 + R_q
                        p = c.p
                        smp = np.random.default_rng(p).integers(0, n, size=64)
                        _, _, (_, Rq) = eng.proj_garble(seed, p, p, [(v * v + 1) % p for v in range(p)], [0], [0], [0])
                        o0 = out0.cpu().numpy().view(np.uint64)
                        ov = outv.cpu().numpy().view(np.uint64)
                        for i in smp.tolist():
                            want = label_add(int(o0[i, 0]) | (int(o0[i, 1]) << 64), Rq, p)
                            assert (int(ov[i, 0]) | (int(ov[i, 1]) << 64)) == want, ("t_proj sweep mismatch", p, i)
                    Ng = N * world if world > 1 else N
                    grows = sum(Ng * p for p in PR[:k])
                    erows = Ng * k
                    gbytes = sum(Ng * (16 * p + 16 + 16 + 16) for p in PR[:k])  # rows + in + out0 + ids
                    ebytes = Ng * k * (16 + 16 + 16 + 8)                       # row + in + out + id
                    line = {"sweep": "tproj", "labels": N, "k": k, "n_gpus": world,
                            "label_ops_per_s": (grows + erows) / (tg + te), "seconds": tg + te,
                            "garble_rows_per_s": grows / tg, "eval_rows_per_s": erows / te,
                            "garble_s": tg, "eval_s": te, "garble_GBps": gbytes / tg / 1e9,
                            "eval_GBps": ebytes / te / 1e9,
                            "check": "eval(base label) == out0 + R_q on 64 sampled gates per lane",
                            "workload": "N independent t_proj gates per CRT lane p_i -> p_i, phi(a) = a^2+1 mod p "
                                        "(bench_main.cpp:40-74), device-resident inputs"}
                    del rows, out0, outv, lab
                    torch.cuda.empty_cache()
                else:
                    g = eng.model("dense1024", 0, k)
                    info = g.info
                    B = max(1, N // 1024)
                    a, b = shard_range(B, world, rank)
                    B = max(1, b - a)
                    seeds = b"".join(int(0x5EED0000 + a + i).to_bytes(16, "big") for i in range(B))
                    P = 1
                    for p in PR[:k]:
                        P *= p
                    lim = min(7, P // 2 - 1)  # encodable inputs (outputs may wrap mod P: throughput only)
                    x = np.random.default_rng(k).integers(-lim, lim + 1, size=(B, 1024))
                    eng.infer(g, seeds, x)  # warm-up at the timed batch: workspace allocated once
                    eng.profile(True)
                    sec, wall, _ = timed(lambda: eng.infer(g, seeds, x))
                    prof = eng.profile_read()
                    eng.profile(False)
                    lin_ms = max_over_ranks(prof.get("linear", (0.0, 0))[0])
                    B = B * world  # whole-job inferences (equal shards)
                    label_macs = 2 * B * 1024 * 1024 * k  # garble + eval passes
                    line = {"sweep": "linear", "labels": B * 1024, "k": k, "n_gpus": world, "inferences": B,
                            "label_macs_per_s_kernel": label_macs / (lin_ms / 1e3) if lin_ms else None,
                            "digit_macs_per_s_kernel": 2 * B * info.linear_macs / (lin_ms / 1e3) if lin_ms else None,
                            "int8_ops_per_s_kernel": 4 * B * info.linear_macs / (lin_ms / 1e3) if lin_ms else None,
                            "linear_kernel_ms": lin_ms, "end_to_end_s": sec,
                            "label_macs_per_s_e2e": label_macs / sec}
                    if lin_ms:
                        _, _, i8, i8_src = measured_peaks()
                        ach = 4 * B * info.linear_macs / (lin_ms / 1e3) / 1e12
                        line["roofline"] = {"bound": "tensor", "achieved": ach, "peak": i8, "unit": "TOPS (int8)",
                                            "frac": ach / i8, "peak_source": i8_src,
                                            "kernel": "tc_linear_kernel (digit rows, tcgen05.mma kind::i8)"}
                        pk = json.load(open(os.path.join(ROOT, "profiles", "int8_peak.json"))).get("tcgen05_issue_peak")
                        if pk:  # the tensor pipe's own ceiling (back-to-back MMAs), beside the cuBLASLt yardstick
                            line["roofline"]["frac_of_mma_issue_peak"] = ach / pk["tops"]
                            line["roofline"]["mma_issue_peak"] = pk["tops"]
                        tp = os.path.join(ROOT, "profiles", "tc_dense_pipe.json")
                        if os.path.exists(tp):  # ncu of the same kernel (k = 8, 4096 inferences, one pass)
                            tj = json.load(open(tp))
                            line["roofline"]["tensor_pipe_ncu"] = {
                                key: tj.get(key) for key in ("tensor_pipe_active_pct", "imma_subpipe_inst_pct",
                                                             "issue_active_pct", "source")}
                if rank == 0:
                    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


SUM_N = [128, 80, 55, 45, 37, 34, 31, 30, 28, 26, 25, 24, 23, 23, 23, 22]  # digits per label, primes 2..53


def _ndig(m):
    """n_digits (label.cpp:15-64): the most base-m digits whose range fits 128 bits."""
    n, v = 0, 1
    while v * m <= 1 << 128:
        v *= m
        n += 1
    return n


def label_add(a: int, b: int, m: int) -> int:
    """compress(decompress_mod(a) + decompress_mod(b)) mod m, digit-wise
    (label.cpp:83-219), for the sweep's sampled property check."""
    n = _ndig(m)
    mod = m ** n
    a, b = a % mod if mod < 1 << 128 else a, b % mod if mod < 1 << 128 else b
    out, pw = 0, 1
    for _ in range(n):
        out += ((a % m + b % m) % m) * pw
        a, b, pw = a // m, b // m, pw * m
    return out


def measured_peaks():
    """HBM GB/s (driver-measured, MEASURED_PEAKS.json) and the int8
    tensor-core peak measured by scripts/int8_peak.py (profiles/int8_peak.json)."""
    hbm, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        hbm, hbm_src = float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    i8, i8_src = 4500.0, "nominal B200 dense int8 (no measured int8 peak)"
    p = os.path.join(ROOT, "profiles", "int8_peak.json")
    if os.path.exists(p):
        j = json.load(open(p))
        i8, i8_src = float(j["tops"]), f"measured: {j.get('how', 'scripts/int8_peak.py')}"
    return hbm, hbm_src, i8, i8_src


def roofline_fields(args, info, B, ms, prof):
    """Roofline of the dominant kernel + every kernel kind of the step.

    Algorithmic bytes per activation element: garbling writes
    16 B per garbled row (uc_cts rows) and reads + writes the element's u8
    label bundle (2 * sum n_p); evaluation reads 16 B per decrypted row
    (eval_rows) plus the same label I/O.  Linear lanes: 2 ops per digit-MAC,
    K * units * sum n_p per pass (linear_macs), garble + eval passes."""
    hbm, hbm_src, i8, i8_src = measured_peaks()
    sum_n = sum(SUM_N[: args.k])
    steps = args.steps
    elems = info.relu_elements * B  # activation elements per step
    out = {}

    def per_launch(kind):
        t, n = prof.get(kind, (0.0, 0))
        return (t / n if n else 0.0), (n / steps if n else 0.0)

    for kind, rows in (("act_garble", info.act_uc_cts), ("act_eval", info.act_eval_rows)):
        t_launch, launches = per_launch(kind)
        if not launches:
            continue
        bpe = 16 * rows + 2 * sum_n
        byts = bpe * elems / launches
        ach = byts / (t_launch / 1e3) / 1e9
        out[kind] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                     "bytes_per_element": bpe, "elements_per_launch": elems / launches,
                     "kernel_ms_per_step": prof[kind][0] / steps,
                     "share_of_step": prof[kind][0] / steps / (ms / steps)}
    t_launch, launches = per_launch("linear")
    if launches and info.linear_macs:
        ops = 2 * 2 * info.linear_macs * B  # garble + eval passes, 2 ops per digit-MAC
        tops = ops / (prof["linear"][0] / steps / 1e3) / 1e12
        out["linear"] = {"bound": "tensor", "achieved": tops, "peak": i8, "unit": "TOPS (int8)", "frac": tops / i8,
                         "peak_source": i8_src, "digit_macs_per_inference_pass": int(info.linear_macs),
                         "kernel_ms_per_step": prof["linear"][0] / steps,
                         "share_of_step": prof["linear"][0] / steps / (ms / steps)}
    for kind in ("setup", "priv_garble", "priv_eval", "encode", "decode", "misc"):
        t, n = prof.get(kind, (0.0, 0))
        if n:
            out[kind] = {"kernel_ms_per_step": t / steps, "share_of_step": t / steps / (ms / steps),
                         "launches_per_step": n / steps}
    head = dict(out.get("act_garble", {}))
    traffic, issue = None, {}
    tp = os.path.join(ROOT, "profiles", "act_garble_traffic.json")
    # the ncu capture is of the headline launch (LeNet-5, k = 8, batch 64): other configs get no traffic figure
    if os.path.exists(tp) and (args.model, args.k, args.batch, args.private) == (MODEL, K, 64, False):
        tj = json.load(open(tp))
        traffic = tj.get("dram_bytes_per_launch")
        issue = {k: tj[k] for k in ("issue_active_frac", "alu_pipe_frac", "warps_active_per_sm",
                                    "warp_instructions_per_launch", "instructions_per_garbled_row") if k in tj}
    roof = {"bound": "hbm", "achieved": head.get("achieved", 0.0), "peak": hbm, "unit": "GB/s",
            "frac": head.get("frac"), "traffic": traffic, "kernel": "act_kernel<garble> (ReLU gadget tape)",
            "peak_source": hbm_src, "bytes_per_element": head.get("bytes_per_element"),
            "kernel_ms_per_step": head.get("kernel_ms_per_step"), "kernel_share_of_step": head.get("share_of_step"),
            "issue_roofline_ncu": issue or None,
            "note": "integer-issue bound (AES T-tables + base-m label codec, SURVEY 8(d) honest note): the HBM "
                    "fraction is small by construction; issue_roofline_ncu (ncu issue-active, ALU pipe, "
                    "instructions per garbled row) is its real roofline"}
    return {"roofline": roof, "rooflines": out}


def launch_ranks(args):
    """--gpus N without a launcher: run this script under torchrun, one rank
    per GPU on 127.0.0.1 (the driver's own launch line), and relay rank 0's
    JSON line.  NCCL's INIT log (communicator + nranks) goes to stderr."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    if not args.emulate:
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def output_checksum(out: np.ndarray) -> int:
    """Order-sensitive digest of decoded outputs (verifies the all-gather)."""
    v = np.ascontiguousarray(out, np.int64).view(np.uint64).astype(object)
    h = 0
    for x in v.ravel().tolist():
        h = (h * 1000003 + x) % ((1 << 61) - 1)
    return h


def run_ours(args, rank, world, local):
    """The product path on this rank's GPU: garble + garble_inputs + evaluate
    + decode_outputs of args.batch fresh inferences per step through
    dashgpu_infer; decoded outputs all-gathered over NCCL once per step.
    --emulate (tests only): the CPU emulation of the device code, gloo and
    wall-clock timing, so the multi-rank launcher is testable without a GPU."""
    import torch
    import torch.distributed as dist

    from paper_2302_06361_b200.engine import Dash

    emu = args.emulate
    if emu:
        dev = torch.device("cpu")
        if world > 1:
            dist.init_process_group("gloo")
        eng = Dash(lib_path=os.path.join(ROOT, "tests", "emu", "libdashemu.so"), emulation=True)
        stream = None
    else:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        if world > 1:
            dist.init_process_group("nccl", device_id=dev)
        stream = torch.cuda.current_stream()
        eng = Dash(local)
        eng.set_stream(stream.cuda_stream)
    g = eng.model(args.model, SEED, args.k, private=args.private)
    info = g.info
    B = args.batch
    n_in, n_out = info.n_in, info.n_out
    rng = np.random.default_rng(1234 + rank)
    host_x = rng.integers(-7, 8, size=(B, n_in)).astype(np.int64)
    dev_x = torch.from_numpy(host_x).to(dev)
    dev_out = torch.zeros((B, n_out), dtype=torch.int64, device=dev)
    steps_seeds = [seeds_for(s, rank, world, B) for s in range(args.warmup + args.steps)]
    dev_seeds = [torch.frombuffer(bytearray(s), dtype=torch.uint8).to(dev) for s in steps_seeds]
    gathered = torch.zeros((world * B, n_out), dtype=torch.int64, device=dev)

    def sync():
        if not emu:
            torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        sync()

    class Timer:
        def __enter__(self):
            barrier()
            if emu:
                self.t0 = time.perf_counter()
            else:
                self.a, self.b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                self.a.record(stream)
            return self

        def __exit__(self, *exc):
            if emu:
                barrier()
                self.ms = 1e3 * (time.perf_counter() - self.t0)
            else:
                self.b.record(stream)
                barrier()
                self.ms = self.a.elapsed_time(self.b)
            t = torch.tensor([self.ms], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max over ranks
            self.ms = float(t.item())

    def step_device(i):
        if emu:
            out, _ = eng.infer(g, steps_seeds[i], host_x)
            dev_out.copy_(torch.from_numpy(out))
        else:
            eng.infer(g, dev_seeds[i].data_ptr(), dev_x.data_ptr(), (dev_out.data_ptr(), B), on_device=True)
        if world > 1:
            dist.all_gather_into_tensor(gathered, dev_out)

    # ---- value: HBM-resident inputs ----
    for i in range(args.warmup):
        step_device(i)
    with ClockSampler(local) if not emu else _Null() as clk:
        with Timer() as tv:
            for i in range(args.steps):
                step_device(args.warmup + i)
    ms = tv.ms
    value = world * B * args.steps / (ms / 1e3)
    # the all-gather of the last step must hold every rank's own decode
    local_sum = torch.tensor([output_checksum(dev_out.cpu().numpy())], dtype=torch.int64, device=dev)
    sums = [torch.zeros_like(local_sum) for _ in range(world)]
    if world > 1:
        dist.all_gather(sums, local_sum)
    else:
        sums = [local_sum]
        gathered.copy_(dev_out)
    gat = gathered.cpu().numpy()
    gather_ok = all(output_checksum(gat[r * B:(r + 1) * B]) == int(sums[r].item()) for r in range(world))
    gather_ok = gather_ok and (gat[rank * B:(rank + 1) * B] == dev_out.cpu().numpy()).all()
    # per-kernel CUDA events (kernels_ms_per_step, roofline) from a second
    # pass of the same steps: the event records cost host time per launch,
    # which a latency-bound small step would otherwise count in `value`
    prof = {}
    if not emu:
        eng.profile(True)
        for i in range(args.steps):
            step_device(args.warmup + i)
        barrier()
        prof = eng.profile_read()
        eng.profile(False)

    # ---- e2e: host buffers through the C ABI (dashgpu_infer) ----
    h2d = d2h = sub_batches = layerwise = 0
    with Timer() as te:
        for i in range(args.steps):
            out_host, tm = eng.infer(g, steps_seeds[args.warmup + i], host_x)
            h2d, d2h = tm.h2d_bytes, tm.d2h_bytes
            sub_batches, layerwise = tm.sub_batches, tm.layerwise
            if world > 1:
                dist.all_gather_into_tensor(gathered, torch.from_numpy(out_host).to(dev))
    e2e = world * B * args.steps / (te.ms / 1e3)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    line = {
        "metric": "garbled inferences/sec (garble+eval)",
        "value": value,
        "unit": "inferences/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": f"{args.model}{' (private weights)' if args.private else ''} "
                               f"({WORKLOADS.get(args.model, 'single-layer sweep')}) k={args.k}, "
                               f"synthetic inputs U[-7,7], batch {B} per GPU, fresh seed per inference per step",
                   "global_batch": world * B, "inferences_per_gpu": B, "parallelism": f"inference-sharded x{world}",
                   "l2": "per-step garbled tables (%.1f GB) exceed L2; no flush needed" % (info.cts * 16 * B / 1e9),
                   "ciphertexts_per_inference": info.cts, "relu_elements_per_inference": info.relu_elements,
                   "sub_batches_per_step": int(sub_batches),
                   "schedule": "layer-windowed" if layerwise else "whole GC per sub-batch"},
        "gather": {"collective": "all_gather of decoded outputs (int64) once per step",
                   "bytes_per_step": world * B * n_out * 8, "verified": bool(gather_ok)},
        "e2e": {"value": e2e, "unit": "inferences/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
    }
    if emu:
        line["emulated"] = "CPU emulation of the device code (tests only): not a measurement"
    else:
        line.update(roofline_fields(args, info, B, ms, prof))
        cpu = None
        sample = args.cpu_sample or min(B, max(8, os.cpu_count() or 8))
        try:
            if world > 1:  # the CPU baseline is an N = 1 figure (taken on rank 0 of a 1-GPU run)
                cpu = {"value": None, "unit": "inferences/s", "cores": os.cpu_count(), "kind": "skipped",
                       "sample": "reported by the N = 1 run only"}
            elif not args.no_cpu:
                cpu = cpu_baseline(reference_circuit(args.model, args.k), n_in, n_out, sample)
        except (Exception, SystemExit) as e:  # the CPU baseline must not hide the GPU line
            cpu = {"value": None, "unit": "inferences/s", "cores": os.cpu_count(), "kind": "unavailable",
                   "sample": str(e)[:200]}
        line["cpu_baseline"] = cpu
        line["clocks"] = clk.summary()
        line["gpu_launches"] = int(sum(v[1] for v in prof.values()))
        line["kernels_ms_per_step"] = {k: v[0] / args.steps for k, v in prof.items() if v[1]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        sys.exit(launch_ranks(args))
    if args.sweep:
        run_sweep(args)
        return
    MODEL_NAME[0] = args.model
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
