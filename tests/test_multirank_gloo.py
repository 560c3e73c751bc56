"""Multi-rank host logic on CPU (gloo, world_size 2): the sharding the library uses (ddks_shard_range, a
host-only C-ABI call) and the combine semantics it implements with NCCL — all-reduce(max) of num, then
all-reduce(min) of the argmax candidates for ddks_stat; contiguous item shards + all-gather for batch and
permutation calls — reproduce the single-rank oracle result exactly. Per-rank partial results come from the
oracle restricted to the rank's shard (there is no GPU here); on a GPU box the same shards run in k_count."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2106_13706_b200 import ddks as K
        from paper_2106_13706_b200 import inputs as I

        out = {}
        # ---- ddks_stat: origins sharded, max + argmax combine
        for seed, (n_P, n_Q, d, kind) in enumerate([(37, 41, 3, "grid"), (200, 150, 5, "mixed"), (1, 2, 2, "normal")]):
            P, Q = I.random_pair(700 + seed, n_P, n_Q, d, kind)
            N = n_P + n_Q
            b, e = K.ddks_shard_range(N, world, rank)
            per = O.per_origin(P, Q, b, e) if e > b else np.zeros(0, np.uint64)
            local = int(per.max()) if per.size else 0
            t = torch.tensor([local], dtype=torch.int64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            num = int(t.item())
            cand = b + int(np.argmax(per == num)) if per.size and (per == num).any() else 2**62
            a = torch.tensor([cand], dtype=torch.int64)
            dist.all_reduce(a, op=dist.ReduceOp.MIN)
            out[f"stat{seed}"] = (num, int(a.item()))
        # ---- ddks_stat_batch: items sharded, all-gather (padded to the largest shard)
        rng = np.random.default_rng(3)
        B = 5
        Pb = rng.integers(0, 4, (B, 9, 3)).astype(np.float32)
        Qb = rng.integers(0, 4, (B, 8, 3)).astype(np.float32)
        b, e = K.ddks_shard_range(B, world, rank)
        b0, e0 = K.ddks_shard_range(B, world, 0)
        chunk = e0 - b0
        mine = np.zeros(chunk, np.int64)
        if e > b:
            mine[: e - b] = O.batch(Pb[b:e], Qb[b:e]).astype(np.int64)
        gathered = [torch.zeros(chunk, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(mine))
        full = []
        for r in range(world):
            rb, re = K.ddks_shard_range(B, world, r)
            full += gathered[r][: re - rb].tolist()
        out["batch"] = full
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_combine_equals_single_rank(world):
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2106_13706_b200 import inputs as I

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for seed, (n_P, n_Q, d, kind) in enumerate([(37, 41, 3, "grid"), (200, 150, 5, "mixed"), (1, 2, 2, "normal")]):
        P, Q = I.random_pair(700 + seed, n_P, n_Q, d, kind)
        num, den, D, arg = O.ddks(P, Q)
        for r in range(world):
            assert res[r][f"stat{seed}"] == (num, arg)
    rng = np.random.default_rng(3)
    Pb = rng.integers(0, 4, (5, 9, 3)).astype(np.float32)
    Qb = rng.integers(0, 4, (5, 8, 3)).astype(np.float32)
    want = O.batch(Pb, Qb).tolist()
    for r in range(world):
        assert res[r]["batch"] == want


def test_bench_reference_arm_under_torchrun_cpu():
    # the driver launches `--impl reference` with torchrun for N > 1: rank 0 prints one JSON line, others exit 0
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--workload", "C1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["value"] > 0 and j["cpu_baseline"]["kind"] == "oracle"
    assert j["e2e"]["h2d_bytes_per_step"] == 0
