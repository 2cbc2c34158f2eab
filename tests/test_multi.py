"""N>1 path on CPU: two gloo ranks shard a batch of inferences, each garbles /
evaluates its shard (CPU emulation of the device code), and the decoded
outputs are all-gathered; the result must equal one process doing the whole
batch.  On the GPU box the same code path runs with NCCL (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import EMU_LIB, ROOT
from paper_2302_06361_b200.shard import shard_range, step_seeds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, out_path):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2302_06361_b200.engine import Dash
    from paper_2302_06361_b200.shard import gather_outputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = Dash(lib_path=EMU_LIB, emulation=True)
    g = eng.model("model_tiny", 1000, 8)
    seeds = step_seeds(0, B)
    a, b = shard_range(B, world, rank)
    x = np.stack([g.random_input(4000 + i) for i in range(a, b)])
    out, _ = eng.infer(g, b"".join(seeds[a:b]), x)
    full = gather_outputs(out, B, g.info.n_out)
    if rank == 0:
        np.save(out_path, full)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover_batch():
    for B in (1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            rs = [shard_range(B, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))


@pytest.mark.skipif(not os.path.exists(EMU_LIB), reason="emulation library not built")
def test_two_rank_gloo_gather_equals_single_process(tmp_path, emu):
    B = 5
    out_path = str(tmp_path / "gathered.npy")
    mp.spawn(_worker, args=(2, _free_port(), B, out_path), nprocs=2, join=True)
    gathered = np.load(out_path)
    g = emu.model("model_tiny", 1000, 8)
    x = np.stack([g.random_input(4000 + i) for i in range(B)])
    single, _ = emu.infer(g, b"".join(step_seeds(0, B)), x)
    assert gathered.shape == single.shape
    assert (gathered == single).all()


def _stream_worker(rank, world, port, out_path):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2302_06361_b200.engine import Dash

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = Dash(lib_path=EMU_LIB, emulation=True)
    g = eng.model("relu1000", 0, 3)
    x = np.random.default_rng(2).integers(-14, 15, size=(1, 1000))
    a, b = shard_range(1000, world, rank)
    out, _, _ = eng.infer_stream(g, int(7).to_bytes(16, "big"), x, 256, u_range=(a, b))
    mine = torch.zeros(1000, dtype=torch.int64)
    mine[a:b] = torch.from_numpy(out[0, a:b])
    dist.all_reduce(mine)  # disjoint shards: the sum is the concatenation
    if rank == 0:
        np.save(out_path, mine.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not os.path.exists(EMU_LIB), reason="emulation library not built")
def test_two_rank_element_sharded_layer_equals_single_process(tmp_path, emu):
    # an activation layer shards by element range with no exchange
    out_path = str(tmp_path / "layer.npy")
    mp.spawn(_stream_worker, args=(2, _free_port(), out_path), nprocs=2, join=True)
    got = np.load(out_path)
    g = emu.model("relu1000", 0, 3)
    x = np.random.default_rng(2).integers(-14, 15, size=(1, 1000))
    single, _, _ = emu.infer_stream(g, int(7).to_bytes(16, "big"), x, 256)
    assert (got == single[0]).all()
    assert (single[0] == np.maximum(x[0], 0)).all()


@pytest.mark.skipif(not os.path.exists(EMU_LIB), reason="emulation library not built")
def test_bench_launches_ranks_itself_and_verifies_the_gather():
    """bench.py --gpus 2 with no launcher spawns two ranks itself (torchrun on
    127.0.0.1), shards the batch, all-gathers the decoded outputs and checks
    the gathered shards against each rank's own decode.  --emulate swaps the
    GPU for the CPU emulation and NCCL for gloo; the launcher is the same."""
    import json
    import subprocess
    import sys

    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--emulate", "--model", "model_tiny",
           "--batch", "3", "--steps", "2", "--warmup", "1", "--no-cpu"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 6
    assert d["gather"]["verified"] is True
    assert d["value"] > 0 and d["e2e"]["value"] > 0
