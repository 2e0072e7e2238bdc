#!/usr/bin/env python
"""Benchmark of the TIDE draft-training hot path (BASELINE.json metric:
"draft-train tokens/sec at 1/2/4/8 B200 + % bf16 tensor peak vs host-CPU ref").

One step = one optimiser step of the EAGLE-3 style draft head over one
micro-batch of synthetic captured hidden states per rank (config C2:
Llama-3.1-8B shape, H 4096, V 128256, S 2048, B 4 -> 8192 positions per rank),
forward + vocabulary-chunked LM-head CE + backward + (NCCL all-reduce) + AdamW.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints one JSON line (rank 0).  `value` is device-timed with inputs resident
in the HBM signal ring; `e2e` is the same metric through the C ABI with the
step's captured states copied from pinned host memory every step.  The
reference arm (--impl reference) times the CPU restatement in oracle/ (the
reference ships no trainer, SPEC.md:8 / SPEC.md:442) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# NCCL communicator-init lines (rank / nranks / transport, NVLS) go to stderr,
# where the driver can count the ranks; stdout stays the one JSON line of the
# contract (NCCL's default debug sink is stdout)
os.environ.setdefault("NCCL_DEBUG", "INFO")
os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

WORKLOAD = "C2"
SEED = 20260217


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=WORKLOAD)
    ap.add_argument("--ttt", type=int, default=1,
                    help="EAGLE-3 training-time-test unroll passes per step (1 = the headline "
                         "single-pass step)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling: fixed global batch of sequences split over the ranks "
                         "(0 = weak scaling, the config's per-rank micro-batch)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ce-probe", action="store_true",
                    help="skip the logit-free (recompute) LM-head backward probe leg")
    ap.add_argument("--cpu-sample-seq", type=int, default=256,
                    help="positions in the bounded CPU sample (one sequence)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=d.get("hbm_gbs", 6650.0), bf16=d.get("bf16_tflops", 1590.0),
                    bf16_sustained=d.get("bf16_tflops_sustained", 1400.0), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sustained=1400.0, src="fallback")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_rank{index}.csv"

    def start(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            # nvidia-smi takes a few hundred ms to start: wait for its first
            # sample so even a short timed region is covered
            t0 = time.time()
            while time.time() - t0 < 5 and self.proc.poll() is None:
                if self.path.stat().st_size > 0:
                    break
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = [l.split(",") for l in self.path.read_text().splitlines() if l.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                s = float(r[1])
                mx = max(mx, float(r[2]))
                if float(r[3]) > 200:  # under load
                    sm.append(s)
                for i, n in enumerate(names):
                    if r[5 + i].strip().lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        if not sm:
            sm = [float(r[1]) for r in rows if len(r) > 1 and r[1].strip().replace(".", "").isdigit()]
        return dict(sm_mhz=statistics.median(sm) if sm else None, sm_max_mhz=mx or None,
                    reasons=sorted(reasons), samples=len(rows))


def ncu_traffic(config):
    """DRAM bytes (read + write) per GEMM launch, averaged over every GEMM
    launch of one step like `achieved` -- from the committed ncu metric capture
    of this workload (profiles/r02_step_ncu_<config>.json, made by
    scripts/ncu_r02.sh; ncu cannot run inside a timed bench), or None."""
    p = ROOT / "profiles" / f"r02_step_ncu_{config}.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        g = d["gemms"]
        dram = sum(x["dram_gb"] for x in g) * 1e9
        alg = sum(x["algorithmic_gb"] for x in g) * 1e9
        return dict(dram_bytes_per_launch=round(dram / len(g)), launches=len(g),
                    dram_over_algorithmic=round(dram / alg, 3),
                    source=f"profiles/{p.name} (ncu --metrics dram__bytes_read.sum,"
                           "dram__bytes_write.sum over one step's GEMM launches; "
                           "scripts/ncu_r02.sh)")
    except Exception:
        return None


def cpu_sample(cfg, seq, threads_note=True):
    """Time one oracle step (the CPU restatement) on a bounded sample: one
    captured sequence of `seq` positions at the workload's model shape."""
    import numpy as np
    import oracle
    K = cfg.get("ttt_steps", 1)
    shp = oracle.make_shape(cfg["hidden"], cfg["vocab"], seq, cfg["n_heads"], cfg["n_kv_heads"],
                            cfg["head_dim"], cfg["ffn"], 1, eps=cfg["rms_eps"],
                            theta=cfg["rope_theta"], ttt=K)
    P = oracle.init_params(shp, SEED)
    E = oracle.init_embedding(shp, SEED)
    cap = oracle.synth_capture(SEED, 0, seq + 1 + K, cfg["vocab"], cfg["hidden"])
    F, u, y, m = oracle.gather_batch(shp, [(cap["ids"], cap["features"])])
    Mst, Vst = np.zeros_like(P), np.zeros_like(P)
    return shp, P, E, (F, u, y, m), Mst, Vst


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from paper_2602_05145_b200 import api
    cfg = workload_cfg(args, api)
    seq = args.cpu_sample_seq
    shp, P, E, batch, Mst, Vst = cpu_sample(cfg, seq)
    hp = [1e-4, 0.9, 0.95, 1e-8, 0.0]
    steps = max(1, min(args.steps, 5))
    warm = max(0, min(args.warmup, 1))
    for k in range(warm):
        oracle.train_step(shp, hp, k + 1, P, Mst, Vst, E, *batch)
    t0 = time.perf_counter()
    for k in range(steps):
        oracle.train_step(shp, hp, warm + k + 1, P, Mst, Vst, E, *batch)
    dt = time.perf_counter() - t0
    tps = steps * seq / dt
    conf = config_block(args, cfg)
    # what this arm actually times: one sequence of `seq` positions per step
    # at the workload's model shape (the whole workload would take hours)
    conf.update(micro_batch=1, seq_len=seq, global_batch=1, tokens_per_rank_step=seq,
                workload_micro_batch=cfg["micro_batch"], workload_seq_len=cfg["seq_len"],
                parallelism="host CPU (rank 0 only)")
    line = dict(impl="reference", metric="draft-train tokens/sec", value=round(tps, 3),
                unit="tokens/s", n_gpus=args.gpus, steps=steps, warmup=warm,
                ms_per_step=round(1e3 * dt / steps, 1), higher_is_better=True,
                scaling=scaling_of(args), vs_baseline=None, dtype="f32 (bf16-rounded operands)", data="synthetic",
                config=conf, host_cpu=cpu_model(),
                cpu_baseline=dict(value=round(tps, 3), unit="tokens/s", cores=oracle.num_threads(),
                                  kind="port",
                                  sample=f"{steps} oracle steps of 1 sequence x {seq} positions at "
                                         f"the {args.config} model shape (full fwd+bwd+AdamW over "
                                         "all trainable params)"),
                e2e=dict(value=round(tps, 3), unit="tokens/s", h2d_bytes_per_step=0,
                         d2h_bytes_per_step=0),
                note="the reference ships no trainer (SPEC.md:8, SPEC.md:442); this arm times the "
                     "repo's C restatement (oracle/) of the same step on the host CPU")
    print(json.dumps(line), flush=True)
    return 0


def cpu_model():
    """lscpu model name and logical core count of the host."""
    name = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for l in out.splitlines():
            if l.startswith("Model name"):
                name = l.split(":", 1)[1].strip()
    except Exception:
        pass
    return dict(model=name, logical_cpus=os.cpu_count())


MODEL_SHAPE = {"C1": "tiny draft head", "C2": "Llama-3.1-8B shape", "C4": "Qwen3-32B shape",
               "C5": "Llama-3.3-70B shape"}


def workload_cfg(args, api):
    cfg = dict(api.CONFIGS[args.config])
    if args.ttt > 1:
        cfg["ttt_steps"] = args.ttt
    if args.global_batch:
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        if args.global_batch % world:
            raise SystemExit(f"--global-batch {args.global_batch} is not divisible by {world} ranks")
        cfg["micro_batch"] = args.global_batch // world
    return cfg


def scaling_of(args):
    return "strong" if args.global_batch else "weak"


def config_block(args, cfg):
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    K = cfg.get("ttt_steps", 1)
    ttt = (f", training-time-test unroll {K} passes (loss weights 0.8^j)" if K > 1 else "")
    name = args.config + (f"-TTT{K}" if K > 1 else "")
    extra = dict(ttt_steps=K) if K > 1 else {}
    return dict(workload=f"{name}: EAGLE-3-style draft head, "
                         f"{MODEL_SHAPE.get(args.config, args.config)} "
                         f"(hidden {cfg['hidden']}, 3-layer feature concat, vocab {cfg['vocab']}, "
                         f"seq {cfg['seq_len']}){ttt}, bf16 GEMMs, synthetic captured hidden states",
                **extra,
                hidden=cfg["hidden"], vocab=cfg["vocab"], seq_len=cfg["seq_len"],
                micro_batch=cfg["micro_batch"], global_batch=cfg["micro_batch"] * world,
                tokens_per_rank_step=cfg["micro_batch"] * cfg["seq_len"],
                parallelism=f"dp{world}",
                l2="inputs larger than L2 (multi-GB per-step working set; no flush needed)")


def run_ours(args):
    import numpy as np
    import torch
    from paper_2602_05145_b200 import _lib, api

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workload_cfg(args, api)
    B, S, H, V = cfg["micro_batch"], cfg["seq_len"], cfg["hidden"], cfg["vocab"]
    T = B * S
    nccl_id = None
    if world > 1:
        obj = [api.DraftTrainer.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    tr = api.DraftTrainer(cfg, seed=SEED, rank=rank, world=world, nccl_id=nccl_id, device=local)
    geom = api.SignalGeometry(H)
    pool_n = 2 * B
    L = S + 1 + cfg.get("ttt_steps", 1)  # every unroll pass fully unmasked
    W = 3 * H
    # ring: the resident pool + the batches of TWO e2e train(job)s (the next
    # job's captured states are appended while the current one trains, <= 16
    # steps and <= 1 GiB each) + one batch of slack; an e2e job may evict the
    # pool (FIFO), which is then re-appended outside the timed regions.  More
    # queued asynchronous DMA than the driver's per-stream work queue holds
    # makes the host block inside the appends until the DMA drains and the
    # steps stop overlapping it (measured at C2: 6 GB jobs read e2e 9% below
    # the device number, 1.6-3.2 GB jobs 2%); with the next job prefetched,
    # at most ~2 GiB are queued.  SPECSIM_BENCH_E2E_JOB overrides the job
    # length (that experiment).
    step_bytes = B * L * (W * 2 + 4)
    per_job = int(os.environ.get("SPECSIM_BENCH_E2E_JOB", "0")) or \
        max(1, min(16, (1 << 30) // step_bytes))
    buf = api.HiddenStateBuffer(geom, capacity_tokens=(pool_n + (2 * per_job + 1) * B) * L,
                                device=local)
    # synthetic captured requests; generated by the library in
    # parallel threads (ctypes releases the GIL)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(pool_n, os.cpu_count() or 4)) as ex:
        caps = list(ex.map(lambda i: api.synth_capture(SEED, rank * 100000 + i, L, V, H),
                           range(pool_n)))
    # pinned host copies of the pool for the end-to-end leg
    pinned = []
    for c in caps:
        t = torch.empty((L, W), dtype=torch.int16, pin_memory=True)
        t.numpy()[:] = c["features"].view(np.int16)
        ids = torch.empty(L, dtype=torch.int32, pin_memory=True)
        ids.numpy()[:] = c["ids"]
        pinned.append((t, ids, c["alpha_s"]))
    # Sample ids are global: rank r's samples are RID * r + p.  train(job) takes
    # the GLOBAL job list (identical on every rank) and shards it: item i of a
    # step's B*world slice goes to rank i mod world (specsim_dp_shard), so rank r
    # must hold exactly the ids at slice positions == r (mod world).
    RID = 10 ** 9
    pool_base = [0]
    next_id = [0]  # same sequence on every rank -> globally known ids

    def load_pool():
        """(re-)append the pool under fresh ids: synchronous, outside timing"""
        pool_base[0] = next_id[0]
        for i, (t, ids, a) in enumerate(pinned):
            _lib.call("specsim_hsbuf_append_packed", buf.h, rank * RID + pool_base[0] + i, a,
                      t.data_ptr(), ids.data_ptr(), L, 0)
        next_id[0] += pool_n

    load_pool()

    def pool_id(r, i):
        return r * RID + pool_base[0] + i % pool_n

    def batch(k):
        """this rank's B pool samples for step k (step / eval calls: local ids)"""
        return [pool_id(rank, k * B + j) for j in range(B)]

    def global_job(steps, id_of):
        return api.global_job(steps, B, world, id_of)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ------------------------------------------------------------ e2e path setup
    # Through the C ABI with the captured states in pinned HOST memory: every
    # step's B samples are appended host -> HBM ring inside the timed region
    # (append_packed mode 2: asynchronous DMA on the buffer's stream) and then
    # train(job) runs the steps; each step waits only for its own samples'
    # copies, so the DMA of later batches overlaps earlier steps.  The job's
    # losses / counters come back to the host.
    h2d = B * L * (W * 2 + 4)
    losses = []

    def append_job(first, n):
        """this rank's captured states of steps first .. first+n-1 (async pinned
        DMA on the buffer's stream); returns the global job's sample ids"""
        base = next_id[0]
        for k in range(n):
            for j in range(B):
                t, idt, a = pinned[((first + k) * B + j) % pool_n]
                _lib.call("specsim_hsbuf_append_packed", buf.h,
                          rank * RID + base + k * B + j, a, t.data_ptr(), idt.data_ptr(), L, 2)
        next_id[0] += n * B
        return global_job(n, lambda r, k, j: r * RID + base + k * B + j)

    def run_e2e(nsteps):
        # jobs of <= per_job steps bound the ring.  Each job's batches are
        # appended (asynchronously, this rank's own samples) BEFORE the previous
        # job trains, so their DMA runs under that job's steps: only the very
        # first batch's copy is exposed.  train(job) returns the job's loss.
        sizes = [min(per_job, nsteps - d) for d in range(0, nsteps, per_job)]
        firsts = [sum(sizes[:i]) for i in range(len(sizes))]
        if os.environ.get("SPECSIM_BENCH_E2E_PROBE") == "resident":
            # diagnostic only: the same job structure on the resident pool (no
            # host -> HBM copies), to separate the DMA from the job structure
            for i in range(len(sizes)):
                job = global_job(sizes[i], lambda r, k, j, o=firsts[i]: pool_id(r, (o + k) * B + j))
                losses.append(tr.train(buf, job, [], epochs=1).mean_loss)
            return
        pending = append_job(firsts[0], sizes[0])
        for i in range(len(sizes)):
            nxt = append_job(firsts[i + 1], sizes[i + 1]) if i + 1 < len(sizes) else None
            o = tr.train(buf, pending, [], epochs=1)
            losses.append(o.mean_loss)
            pending = nxt

    # ------------------------------------------------------------ timed legs
    # Device-timed leg: K optimiser steps through train(job) -- the entry point
    # the reference's maybe_trigger_training calls -- with the
    # captured states already resident in the HBM ring; train() enqueues the
    # steps back-to-back (one CUDA graph launch each); timed with CUDA events on
    # the trainer's stream.  End-to-end leg: the same K steps through the
    # pinned-host appends above, host wall clock.  The e2e leg runs between
    # the two halves of the device-timed leg (value, e2e, value) so both sample
    # the same point of the power / clock ramp of a short run.
    valid = 0
    for k in range(args.warmup):
        valid = int(tr.step(buf, batch(k))["valid_tokens"])
    if not args.no_e2e:
        run_e2e(max(1, args.warmup))
        load_pool()
    # value leg in two halves around one end-to-end leg of all K steps: both
    # legs centred on the same point of the power / clock ramp, and the e2e
    # leg's unhidden first-batch DMA paid once, as in a single job
    halves = [args.steps] if args.steps < 2 else [args.steps // 2, args.steps - args.steps // 2]
    clocks = ClockSampler(local)
    region_ms, dt_e2e, e2e_dev_ms, launches, done_steps = 0.0, 0.0, 0.0, 0, 0
    value_losses = []
    barrier()
    clocks.start()
    for hi, hs in enumerate(halves):
        job = global_job(hs, lambda r, k, j, o=done_steps:
                         pool_id(r, (args.warmup + o + k) * B + j))
        barrier()
        launches0 = _lib.kernel_launches()
        tr.region_begin()
        out = tr.train(buf, job, [], epochs=1)
        ms = tr.region_end()
        launches += _lib.kernel_launches() - launches0
        region_ms += max_over_ranks(ms)
        value_losses.append(out.mean_loss)
        done_steps += hs
        if hi == 0 and not args.no_e2e:
            barrier()
            t0 = time.perf_counter()
            tr.region_begin()
            run_e2e(args.steps)
            e2e_dev_ms = tr.region_end()
            barrier()
            dt_e2e = max_over_ranks(time.perf_counter() - t0)
            load_pool()
    clk = clocks.stop()
    barrier()
    value = world * T * args.steps / (region_ms / 1e3)
    e2e = None
    if not args.no_e2e:
        e2e = dict(value=round(world * T * args.steps / dt_e2e, 1), unit="tokens/s",
                   h2d_bytes_per_step=h2d, d2h_bytes_per_step=3 * 8,
                   ms_per_step=round(1e3 * dt_e2e / args.steps, 2),
                   device_ms_per_step=round(e2e_dev_ms / args.steps, 3),
                   timing="host wall clock around the async pinned-host appends + train(job) "
                          "of the K steps (jobs of <= 1 GiB of captured states; job i+1's appends "
                          "are issued before job i trains, so its DMA overlaps job i's steps), "
                          "run between the two halves of the device-timed leg, max over ranks")
        # ingest alone (reported separately): one job's worth of
        # pinned-host appends with nothing else running, host wall clock
        n_in = per_job * B
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(n_in):
            t, idt, a = pinned[i % pool_n]
            _lib.call("specsim_hsbuf_append_packed", buf.h, rank * RID + next_id[0] + i, a,
                      t.data_ptr(), idt.data_ptr(), L, 2)
        torch.cuda.synchronize()
        dt_in = time.perf_counter() - t0
        next_id[0] += n_in
        e2e["ingest"] = dict(h2d_GBps=round(n_in * L * (W * 2 + 4) / dt_in / 1e9, 1),
                             tokens_per_s=round(n_in * L / dt_in, 1),
                             sample=f"{n_in} captured requests of {L} tokens appended "
                                    "(append_packed, async pinned DMA), nothing else running")
        load_pool()

    # ------------------------------------------------------------ roofline leg
    # Per-phase device time with CUDA events around every launch (a graph with
    # timestamp nodes).  Measured on the LAST step of back-to-back train(job)
    # jobs -- the same steady-state power / clock regime as the value leg
    # (single synchronous steps leave idle gaps that let the clock recover and
    # would read several % fast).  A first job captures the timing graph.
    n_prof = min(args.steps, 3)
    prof_job = max(4, min(args.steps, 8))
    tr.set_timing(True)
    phase_acc = {p: dict(ms=0.0, flops=0.0, launches=0) for p in api.DraftTrainer.PHASES}
    barrier()
    tr.train(buf, global_job(2, lambda r, k, j: pool_id(r, k * B + j)), [], epochs=1)
    prof_step_ms = 0.0
    for k in range(n_prof):
        job = global_job(prof_job, lambda r, kk, j, o=k: pool_id(r, (o * prof_job + kk) * B + j))
        tr.train(buf, job, [], epochs=1)
        prof_step_ms += max_over_ranks(tr.last_step_ms())
        for p, v in tr.phase_times().items():
            for f in ("ms", "flops", "launches"):
                phase_acc[p][f] += v[f]
    tr.set_timing(False)
    barrier()

    # ------------------------------------------------------------ roofline
    pk = peaks()
    fl = api.gemm_flops_per_token(cfg)
    gemm_ms = phase_acc["gemm"]["ms"] + phase_acc["lm_head_ce"]["ms"]
    gemm_alg = phase_acc["gemm"]["flops"] + phase_acc["lm_head_ce"]["flops"]
    achieved = gemm_alg / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else None
    traffic = ncu_traffic(args.config) if cfg.get("ttt_steps", 1) == 1 else None
    roofline = dict(bound="tensor", kernel="gemm_kernel<tcgen05> (all GEMM launches of the step)",
                    achieved=round(achieved, 1) if achieved else None,
                    peak=pk["bf16_sustained"], unit="TFLOP/s",
                    frac=round(achieved / pk["bf16_sustained"], 4) if achieved else None,
                    peak_source=f"{pk['src']} bf16_tflops_sustained (kernel timed inside a long step)",
                    traffic=traffic.get("dram_bytes_per_launch") if traffic else None,
                    traffic_over_algorithmic=traffic.get("dram_over_algorithmic") if traffic
                    else None,
                    traffic_source=traffic.get("source") if traffic else None,
                    algorithmic="SURVEY §8(d): sum of GEMM FLOPs excluding the CE-backward logit "
                                "recompute, over the summed device time of every GEMM launch "
                                "(recompute time included)",
                    measured=f"CUDA events around every GEMM launch of the last step of "
                             f"{n_prof} back-to-back {prof_job}-step train(job) jobs run right "
                             "after the value leg (steady-state clock, as the value leg)")
    step_ms = region_ms / args.steps
    phases = {p: dict(ms_per_step=round(v["ms"] / n_prof, 3),
                      launches_per_step=v["launches"] // max(1, n_prof))
              for p, v in phase_acc.items()}
    # device time of the profiled (last) steps not inside any timed launch
    # (launch gaps, event nodes, per-step input fetch / result store)
    phases["untimed_gaps"] = dict(
        ms_per_step=round((prof_step_ms - sum(v["ms"] for v in phase_acc.values())) / n_prof, 3),
        launches_per_step=0)
    whole_step_tflops = fl["total"] * T / (step_ms / 1e3) / 1e12

    line = dict(metric="draft-train tokens/sec", value=round(value, 1), unit="tokens/s",
                n_gpus=world, steps=args.steps, warmup=args.warmup,
                ms_per_step=round(step_ms, 3), higher_is_better=True, scaling=scaling_of(args),
                vs_baseline=None, dtype="bf16", data="synthetic (seeded captured hidden states, "
                "random-init draft weights)", config=config_block(args, cfg), e2e=e2e,
                roofline=roofline, gpu_launches=int(launches),
                valid_tokens_per_rank_step=valid,
                whole_step=dict(tflops=round(whole_step_tflops, 1),
                                frac_of_peak=round(whole_step_tflops / pk["bf16_sustained"], 4),
                                gflop_per_token=round(fl["total"] / 1e9, 4)),
                phases=phases,
                loss_mean_value_leg=round(sum(value_losses) / len(value_losses), 4),
                clocks=clk)

    # ------------------------------------------------------------ CE probe
    # north_star (3) asks that full logits never reach HBM.  The default step
    # stores them as fp16 offsets (2 B x T x V) because that beats recomputing
    # them in the backward (DESIGN.md §3 K6, §10); the logit-free path
    # (SPECSIM_CE_RECOMPUTE=1: the CE-backward GEMM recomputes each logit tile
    # in TMEM and writes the bf16 gradient tile directly) is timed here on a
    # second trainer so every bench line reports both.
    if rank == 0 and world == 1 and not args.no_ce_probe:
        try:
            os.environ["SPECSIM_CE_RECOMPUTE"] = "1"
            tr2 = api.DraftTrainer(cfg, seed=SEED, device=local)
            os.environ.pop("SPECSIM_CE_RECOMPUTE")
            # same method as the roofline leg: last step of back-to-back jobs
            tr2.train(buf, global_job(2, lambda r, k, j: pool_id(r, k * B + j)), [], epochs=1)
            tr2.set_timing(True)
            tr2.train(buf, global_job(2, lambda r, k, j: pool_id(r, k * B + j)), [], epochs=1)
            acc, st = 0.0, 0.0
            for k in range(n_prof):
                job = global_job(prof_job, lambda r, kk, j, o=k: pool_id(r, (o * prof_job + kk) * B + j))
                tr2.train(buf, job, [], epochs=1)
                st += tr2.last_step_ms()
                acc += tr2.phase_times()["lm_head_ce"]["ms"]
            tr2.close()
            line["ce_recompute_probe"] = dict(
                lm_head_ce_ms_per_step=round(acc / n_prof, 3), step_ms=round(st / n_prof, 3),
                default_lm_head_ce_ms_per_step=phases["lm_head_ce"]["ms_per_step"],
                note=f"logit-free LM-head + CE backward (no [T, V] logits in HBM); last step of "
                     f"{n_prof} back-to-back {prof_job}-step jobs, phase events on (as the "
                     "default's phases); the default path stores fp16 logit offsets instead "
                     "(DESIGN.md §3 K6)")
        except Exception as e:  # reported, never required
            os.environ.pop("SPECSIM_CE_RECOMPUTE", None)
            line["ce_recompute_probe"] = dict(error=str(e)[:200])

    # ------------------------------------------------------------ CPU baseline
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            seq = args.cpu_sample_seq
            shp, P, E, batch_c, Mst, Vst = cpu_sample(cfg, seq)
            t0 = time.perf_counter()
            oracle.train_step(shp, [1e-4, 0.9, 0.95, 1e-8, 0.0], 1, P, Mst, Vst, E, *batch_c)
            dtc = time.perf_counter() - t0
            line["cpu_baseline"] = dict(
                value=round(seq / dtc, 3), unit="tokens/s", cores=oracle.num_threads(),
                kind="port", host_cpu=cpu_model(),
                sample=f"1 oracle step (fwd+bwd+AdamW, all {args.config} params) on 1 sequence x "
                       f"{seq} positions; {dtc:.1f} s")
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = dict(value=None, unit="tokens/s", cores=os.cpu_count(),
                                        kind="port", sample=f"failed: {e}")
    if rank == 0:
        print(json.dumps(line), flush=True)
    tr.close()
    buf.close()
    if dist:
        dist.destroy_process_group()
    return 0


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(args):
    """--gpus N > 1 without a torchrun environment: re-exec this script under
    torch.distributed.run with N ranks on this node (one per GPU); the exit
    code is the launcher's.  Under torchrun, WORLD_SIZE must equal --gpus."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(ROOT / "bench.py"), *sys.argv[1:]]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1 and args.impl == "ours":
        return launch_ranks(args)
    if world_env is not None and int(world_env) != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}: launch one "
                         "rank per GPU (torchrun --nproc-per-node N ... --gpus N)")
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
