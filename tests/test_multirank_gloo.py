"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the sharding the library uses (ddks_shard_range, a
host-only C-ABI call) and the combine steps it runs after its one NCCL all-gather, driven through the library's
own exported host functions — ddks_combine_records for ddks_stat (one {num, argmax, flags} record per rank; also
the x0-ordered origin shards below), ddks_unpad_items for the padded per-item records of batch, permutation and
batched-significance calls (totals not divisible by the world size, fewer items than ranks); histogram all-reduce(sum) + sharded table +
rank-ordered partial sums for the significance; voxel shards (vdKS) and corner shards (rdKS) with max / min-index
combines — reproduce the single-rank oracle result. Per-rank partial results come from the
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
STAT_CASES = [(37, 41, 3, "grid"), (200, 150, 5, "mixed"), (1, 2, 2, "normal"), (6, 5, 2, "grid")]
BATCH_SIZES = [5, 7, 2, 1]  # totals not divisible by the world size, and fewer items than ranks


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
        # ---- ddks_stat: origins sharded; every rank contributes ONE record {num, argmax candidate, flags} (the library's
        # single all-gather), combined by the library's exported host step ddks_combine_records
        for seed, (n_P, n_Q, d, kind) in enumerate(STAT_CASES):
            P, Q = I.random_pair(700 + seed, n_P, n_Q, d, kind)
            N = n_P + n_Q
            b, e = K.ddks_shard_range(N, world, rank)
            per = O.per_origin(P, Q, b, e) if e > b else np.zeros(0, np.uint64)
            local = int(per.max()) if per.size else 0
            cand = b + int(np.argmax(per == local)) if per.size else -1
            rec = torch.tensor([local, cand, 1 if seed == 2 and rank == world - 1 else 0], dtype=torch.int64)
            recs = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(recs, rec)
            out[f"stat{seed}"] = K.ddks_combine_records([tuple(int(v) for v in r.tolist()) for r in recs])
        # ---- ddks_stat_batch / ddks_permutation_null: items sharded; ONE all-gather of records padded to the largest
        # shard (this rank's nums, then its flags word), unpadded by the library's exported ddks_unpad_items
        rng = np.random.default_rng(3)
        for B in BATCH_SIZES:
            Pb = rng.integers(0, 4, (B, 9, 3)).astype(np.float32)
            Qb = rng.integers(0, 4, (B, 8, 3)).astype(np.float32)
            b, e = K.ddks_shard_range(B, world, rank)
            stride = K.gather_stride(B, world, 2)
            chunk = (stride - 1) // 2
            rec = np.zeros(stride, np.uint64)
            if e > b:
                rec[: e - b] = O.batch(Pb[b:e], Qb[b:e])
                rec[chunk: chunk + e - b] = np.arange(b, e, dtype=np.uint64) * 7  # a second per-item array
            rec[2 * chunk] = 2 if rank == 0 and B == 7 else 0  # flags word
            gathered = [torch.zeros(stride, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(rec.view(np.int64)))
            flat = torch.cat(gathered).numpy().view(np.uint64)
            items, flags = K.ddks_unpad_items(flat, B, world, 2)
            out[f"batch{B}"] = (items[0].tolist(), items[1].tolist(), flags, O.batch(Pb, Qb).tolist())

        # ---- x0-ordered ddks_stat: ranks shard POSITIONS of the x_0 order (ties keep pooled order); each rank's
        # per-origin nums land in a zeroed pooled-order array; max, then argmax over the full array, min over ranks
        P, Q = I.random_pair(733, 90, 70, 4, "grid")
        pooled = np.concatenate([P, Q])
        N = pooled.shape[0]
        order = np.lexsort((np.arange(N), pooled[:, 0]))  # key x_0, then pooled index
        b, e = K.ddks_shard_range(N, world, rank)
        per_full = np.zeros(N, np.uint64)
        for j in range(b, e):
            o = int(order[j])
            per_full[o] = O.per_origin(P, Q, o, o + 1)[0]
        t = torch.tensor([int(per_full.max())], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        num = int(t.item())
        hit = np.nonzero(per_full == num)[0]
        a = torch.tensor([int(hit[0]) if hit.size else 2**62], dtype=torch.int64)
        dist.all_reduce(a, op=dist.ReduceOp.MIN)
        out["x0"] = (num, int(a.item()))

        # ---- ddks_significance: origins sharded -> M_T histogram all-reduce(sum); table entries sharded; partial
        # sums all-gathered and added in rank order
        P, Q = I.random_pair(741, 30, 25, 2, "normal")
        pooled = np.concatenate([P, Q])
        N, n_Q = pooled.shape[0], Q.shape[0]
        b, e = K.ddks_shard_range(N, world, rank)
        MT = O.membership(Q, pooled[b:e]) if e > b else np.zeros((0, 4), np.int64)
        h = torch.from_numpy(np.bincount(MT.ravel(), minlength=n_Q + 1).astype(np.int64))
        dist.all_reduce(h, op=dist.ReduceOp.SUM)
        num = O.ddks(P, Q)[0]
        mb, me = K.ddks_shard_range(n_Q + 1, world, rank)
        part = sum(int(h[m]) * np.log(O.p_le(num, P.shape[0], n_Q, (m + 1.0) / (n_Q + 2.0)))
                   for m in range(mb, me) if int(h[m]) > 0)
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.tensor([float(part)], dtype=torch.float64))
        out["sig"] = (h.tolist(), sum(float(x.item()) for x in parts))

        # ---- ddks_vdks: voxel counts all-reduced, voxels sharded, max combine
        P, Q = I.random_pair(751, 60, 50, 3, "mixed")
        k = 4
        vb, ve = K.ddks_shard_range(k ** 3, world, rank)
        t = torch.tensor([O.vdks(P, Q, k, vb, ve)[0]], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["vdks"] = int(t.item())

        # ---- ddks_rdks: corners sharded, max + first attaining corner
        P, Q = I.random_pair(761, 60, 50, 4, "normal")
        cb, ce = K.ddks_shard_range(5, world, rank)
        r = O.rdks(P, Q, cb, ce)
        t = torch.tensor([r[0]], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        num = int(t.item())
        a = torch.tensor([r[3] if (ce > cb and r[0] == num) else 2**62], dtype=torch.int64)
        dist.all_reduce(a, op=dist.ReduceOp.MIN)
        out["rdks"] = (num, int(a.item()))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
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
    for seed, (n_P, n_Q, d, kind) in enumerate(STAT_CASES):
        P, Q = I.random_pair(700 + seed, n_P, n_Q, d, kind)
        num, den, D, arg = O.ddks(P, Q)
        for r in range(world):
            assert res[r][f"stat{seed}"] == (num, arg, 1 if seed == 2 else 0)
    for B in BATCH_SIZES:
        for r in range(world):
            nums, second, flags, want = res[r][f"batch{B}"]
            assert nums == want and second == [7 * i for i in range(B)]
            assert flags == (2 if B == 7 else 0)
    # x0-ordered sharding == single-rank statistic and argmax
    P, Q = I.random_pair(733, 90, 70, 4, "grid")
    num, den, D, arg = O.ddks(P, Q)
    # significance: the summed histogram is the single-rank one, and the sharded sum of logs matches the oracle
    Ps, Qs = I.random_pair(741, 30, 25, 2, "normal")
    S, lp, _ = O.significance(Ps, Qs)
    pooled = np.concatenate([Ps, Qs])
    h_full = np.bincount(O.membership(Qs, pooled).ravel(), minlength=Qs.shape[0] + 1).tolist()
    for r in range(world):
        assert res[r]["x0"] == (num, arg)
        assert res[r]["sig"][0] == h_full
        assert abs(res[r]["sig"][1] - lp) <= 1e-9 * max(1.0, abs(lp))
        Pv, Qv = I.random_pair(751, 60, 50, 3, "mixed")
        assert res[r]["vdks"] == O.vdks(Pv, Qv, 4)[0]
        Pr, Qr = I.random_pair(761, 60, 50, 4, "normal")
        want_r = O.rdks(Pr, Qr)
        assert res[r]["rdks"] == (want_r[0], want_r[3])


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
