"""Data-parallel path on CPU with world_size 2 (gloo): each rank takes its
shard by the library's sharding rule (specsim_dp_shard, the same rule
DraftTrainer::train uses), runs the oracle step with the globally all-reduced
valid-token count, all-reduces (sums) the gradients and applies AdamW.  The
result must equal the single-process step on the whole global batch — the
property the NCCL path in trainer.cu relies on (loss normalised by the global
sum of masks, gradients summed)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2602_05145_b200 import api

SH = dict(H=64, V=512, S=32, nh=4, nkv=2, hd=16, I=128)
HP = [1e-3, 0.9, 0.95, 1e-8, 0.01]
LENS = [34, 20, 34, 9, 34, 30]  # 6 samples, some short (masked tails)
WORLD, PER_RANK = 2, 2


def samples():
    out = []
    for i, L in enumerate(LENS):
        c = oracle.synth_capture(5, i, L, SH["V"], SH["H"])
        out.append((c["ids"], c["features"]))
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    shp = oracle.make_shape(**SH, B=PER_RANK)
    P = oracle.init_params(shp, 3)
    E = oracle.init_embedding(shp, 3)
    smp = samples()
    Mst, Vst = np.zeros_like(P), np.zeros_like(P)
    results = []
    for step in range(2):  # 6 samples, 4 per global step -> second step is partial
        mine = api.dp_shard(len(LENS), PER_RANK, WORLD, rank, step)
        F, u, y, m = oracle.gather_batch(shp, [smp[i] for i in mine])
        n = torch.tensor([int(m.sum())], dtype=torch.int64)
        dist.all_reduce(n)
        out, g = oracle.train_step(shp, HP, step + 1, P, Mst, Vst, E, F, u, y, m,
                                   global_valid=int(n.item()), update=False)
        gt = torch.from_numpy(g)
        dist.all_reduce(gt)
        loss = torch.tensor([out.loss], dtype=torch.float64)
        dist.all_reduce(loss)
        oracle.adamw(P, Mst, Vst, gt.numpy(), HP, step + 1)
        results.append((float(loss.item()), gt.numpy().copy(), P.copy(), mine))
    if rank == 0:
        q.put(results)
    dist.barrier()
    dist.destroy_process_group()


def test_sharding_rule():
    got = [api.dp_shard(6, 2, 2, r, s) for s in range(2) for r in range(2)]
    assert got == [[0, 2], [1, 3], [4], [5]]
    assert api.dp_shard(3, 4, 1, 0, 0) == [0, 1, 2]
    assert api.dp_shard(10, 2, 4, 3, 1) == [] and api.dp_shard(10, 2, 4, 1, 1) == [9]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_global_job_routes_each_rank_its_own_samples(world):
    """bench.py / callers build ONE global job list; train(job) shards it by
    specsim_dp_shard.  Every rank must get exactly its own B samples per step."""
    B, RID, steps = 4, 10 ** 9, 5
    job = api.global_job(steps, B, world, lambda r, k, j: r * RID + k * B + j)
    for r in range(world):
        for k in range(steps):
            mine = [job[i] for i in api.dp_shard(len(job), B, world, r, k)]
            assert mine == [r * RID + k * B + j for j in range(B)], (world, r, k)


def test_world2_equals_single_process_global_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single process, whole global batch of each step
    shp = oracle.make_shape(**SH, B=PER_RANK * WORLD)
    P = oracle.init_params(shp, 3)
    E = oracle.init_embedding(shp, 3)
    smp = samples()
    Mst, Vst = np.zeros_like(P), np.zeros_like(P)
    for step in range(2):
        batch = smp[step * 4:(step + 1) * 4]
        F, u, y, m = oracle.gather_batch(shp, batch)
        out, g = oracle.train_step(shp, HP, step + 1, P, Mst, Vst, E, F, u, y, m)
        loss_dp, g_dp, P_dp, _ = res[step]
        assert abs(loss_dp - out.loss) < 1e-6 * abs(out.loss)
        assert np.linalg.norm(g_dp - g) / np.linalg.norm(g) < 1e-5
        assert np.abs(P_dp - P).max() < 1e-3 * HP[0] + 1e-7


# ------------------------------------------------------------------ ZeRO-1
@pytest.mark.parametrize("cfg", ["C1", "C2", "C4", "C5"])
def test_dp_buckets_tile_the_registry(cfg):
    """The exchange buckets (specsim_dp_buckets, the trainer's own list) tile
    the flat parameter vector; ZeRO-1 shards of every world size in 1..8 are
    disjoint, complete and 8-element aligned."""
    c = api.CONFIGS[cfg]
    shp = oracle.make_shape(c["hidden"], c["vocab"], c["seq_len"], c["n_heads"], c["n_kv_heads"],
                            c["head_dim"], c["ffn"], 1)
    _, total = oracle.param_layout(shp)
    for world in (1, 2, 4, 8):
        buckets, ok = api.dp_buckets(c, world)
        assert ok, (cfg, world)
        ranges = sorted(buckets)
        assert ranges[0][0] == 0 and sum(n for _, n in ranges) == total
        assert all(a[0] + a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        covered = np.zeros(1 << 16, np.int64)  # coverage count per bucket-local shard slot
        for bk in buckets:
            shards = [api.zero_shard(bk, world, r) for r in range(world)]
            assert shards[0][0] == bk[0] and shards[-1][1] == bk[0] + bk[1]
            assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
            assert all((lo % 8, hi % 8) == (0, 0) for lo, hi in shards)
        del covered
    # 12 ranks do not divide the 64-aligned buckets of C1 into 8-element groups
    assert not api.dp_buckets(api.CONFIGS["C1"], 12)[1]


def _zero_worker(rank, port, q):
    """ZeRO-1 as the trainer runs it: per bucket, reduce-scatter (here: the
    all-reduced sum restricted to the rank's shard), AdamW on the shard only,
    all-gather of the updated shard."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    shp = oracle.make_shape(**SH, B=PER_RANK)
    cfg = dict(hidden=SH["H"], vocab=SH["V"], seq_len=SH["S"], n_heads=SH["nh"],
               n_kv_heads=SH["nkv"], head_dim=SH["hd"], ffn=SH["I"], micro_batch=PER_RANK)
    buckets, ok = api.dp_buckets(cfg, WORLD)
    assert ok
    P = oracle.init_params(shp, 3)
    E = oracle.init_embedding(shp, 3)
    smp = samples()
    Mst, Vst = np.zeros_like(P), np.zeros_like(P)
    results = []
    for step in range(2):
        mine = api.dp_shard(len(LENS), PER_RANK, WORLD, rank, step)
        F, u, y, m = oracle.gather_batch(shp, [smp[i] for i in mine])
        n = torch.tensor([int(m.sum())], dtype=torch.int64)
        dist.all_reduce(n)
        _, g = oracle.train_step(shp, HP, step + 1, P, Mst, Vst, E, F, u, y, m,
                                 global_valid=int(n.item()), update=False)
        for bk in buckets:
            lo, hi = api.zero_shard(bk, WORLD, rank)
            gb = torch.from_numpy(g[bk[0]:bk[0] + bk[1]].copy())
            dist.all_reduce(gb)  # reduce-scatter = the sum, keeping only this rank's shard
            gs = gb.numpy()[lo - bk[0]:hi - bk[0]].copy()
            p, ms, vs = P[lo:hi].copy(), Mst[lo:hi].copy(), Vst[lo:hi].copy()
            oracle.adamw(p, ms, vs, gs, HP, step + 1)
            Mst[lo:hi], Vst[lo:hi] = ms, vs
            parts = [torch.zeros(hi - lo, dtype=torch.float32) for _ in range(WORLD)]
            dist.all_gather(parts, torch.from_numpy(p))
            P[bk[0]:bk[0] + bk[1]] = torch.cat(parts).numpy()
        results.append(P.copy())
    if rank == 0:
        q.put(results)
    dist.barrier()
    dist.destroy_process_group()


def test_world2_zero1_equals_single_process_global_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_zero_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    shp = oracle.make_shape(**SH, B=PER_RANK * WORLD)
    P = oracle.init_params(shp, 3)
    E = oracle.init_embedding(shp, 3)
    smp = samples()
    Mst, Vst = np.zeros_like(P), np.zeros_like(P)
    for step in range(2):
        F, u, y, m = oracle.gather_batch(shp, smp[step * 4:(step + 1) * 4])
        oracle.train_step(shp, HP, step + 1, P, Mst, Vst, E, F, u, y, m)
        assert np.abs(res[step] - P).max() < 1e-3 * HP[0] + 1e-7, step
