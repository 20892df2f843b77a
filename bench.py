#!/usr/bin/env python
"""Headline benchmark: certified inference requests/s for the ResNet-50 model
group (BASELINE.json: configs[1] = C2: 3 replicas, f=1, batch 128, 224x224,
random-init jittered weights, synthetic signed requests).

A step = one ExecutionBatch through the whole hot path: 3 replica forwards
(tcgen05 convs) -> softmax/top-k -> select_quorum + label vote -> result
leaves (request midstates shared by the providers), R roots, attestation
manifest + A root. A request counts as certified when its quorum is
satisfied and all of that is produced.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1 runs under torchrun, one rank per GPU, each rank certifying its own
request stream for its own replica set (weak scaling, no data-path
collective: requests are independent objects); the timed region is
bracketed by barriers and the max over ranks is taken.

--mode replica (N>1): the reference's own deployment shape — an N-replica
group, rank k serving replica assigned_models(N, G, k) (domain.cpp:247-268),
every rank certifying the SAME request stream; replica outputs and R roots
are exchanged with one NCCL all-gather per batch (cg_group_create_dist).
"""
from __future__ import annotations

import argparse
import copy
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "certified inference requests/s (ResNet-50 group) at 1/2/4/8 B200 vs host CPU"
UNIT = "req/s"
SIZE = 224
U = 3 * SIZE * SIZE


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0,
                "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # nvidia-smi takes a moment to produce its first row
            while not self.rows and time.time() - t0 < 5:
                time.sleep(0.05)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for n, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------------ setup
def make_group(ctx, B, seed=0, eps=0.1):
    from paper_2205_15757_b200 import EUCLIDEAN, Model, ModelGroup
    from paper_2205_15757_b200.workload import resnet_group
    files, digs, sds = resnet_group("resnet50", replicas=3, seed=seed, jitter=5e-3)
    models = [Model.load_cnn(ctx, f, d) for f, d in zip(files, digs)]
    grp = ModelGroup(ctx, models, 1, EUCLIDEAN, eps, b"group-0", 1, max_batch=B, topk=5)
    return grp, models, files, digs, sds


C3_EPS = 1.5  # >= sqrt(2): random-init nets of different families do not agree tightly


def make_hetero_group(ctx, B, seed=0, eps=C3_EPS):
    """C3 (BASELINE.json configs[2]): ResNet-50, ResNet-101, VGG-16,
    MobileNetV2, one replica each, f = 1."""
    from paper_2205_15757_b200 import EUCLIDEAN, Model, ModelGroup
    from paper_2205_15757_b200.workload import HETERO_GROUP, hetero_group
    files, digs, sds = hetero_group(HETERO_GROUP, seed=seed)
    models = [Model.load_cnn(ctx, f, d) for f, d in zip(files, digs)]
    grp = ModelGroup(ctx, models, 1, EUCLIDEAN, eps, b"group-0", 1, max_batch=B, topk=5)
    return grp, models, files, digs, sds


def resnet50_gemm_plan(B, R, S=224):
    """(name, FLOPs, compulsory HBM bytes) of each conv GEMM launch of one
    grouped ResNet-50 forward over R replicas, in csrc/cnn.cu ResNet::ops
    order (conv1, per block c1, c2, c3 -- with the projection shortcut fused
    into c3 in the first block of each stage -- fc); same model as
    tools/step_roofline.py."""
    L = []
    px = lambda h: B * h * h  # noqa: E731
    H1, H = S // 2, S // 4
    # conv1: the s2d stem reads the 2-plane space-to-depth image (16 B per
    # plane and grid pixel, ((S + 6) / 2)^2 grid pixels per image)
    G = (S + 6) // 2
    L.append(("conv1", 2 * px(H1) * 64 * 147 * R, B * G * G * 32 + R * px(H1) * 64 * 2))
    cin = 64
    for stage, (w, n) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        for i in range(n):
            s = 2 if (i == 0 and stage > 0) else 1
            Ho, cout = H // s, 4 * w
            L.append(("c1", 2 * px(H) * cin * w * R, R * (px(H) * cin * 2 + px(H) * w * 2)))
            L.append(("c2", 2 * px(Ho) * 9 * w * w * R, R * (px(H) * w * 2 + px(Ho) * w * 2)))
            if i == 0:  # c3 + projection shortcut, one GEMM over K = w + cin
                L.append(("c3+ds", 2 * px(Ho) * (w + cin) * cout * R,
                          R * (px(Ho) * (w + cin) * 2 + px(Ho) * cout * 2)))
            else:
                L.append(("c3", 2 * px(Ho) * w * cout * R,
                          R * (px(Ho) * w * 2 + 2 * px(Ho) * cout * 2)))
            H, cin = Ho, cout
    L.append(("fc", 2 * B * cin * 1000 * R, R * (B * cin * 2 + B * 1000 * 4)))
    return L


def replica_f(n):
    return (n - 1) // 3  # the largest f with n >= 3f + 1 (ClusterConfig::validate)


def make_dist_group(ctx, B, rank, world, seed=0, eps=0.1, N=None):
    """Replica-parallel group of N (default: world) replicas: rank serves
    assigned_models(world, N, rank) (domain.cpp:247-268: one replica per GPU
    when N == world, contiguous chunks otherwise); NCCL communicator from
    rank 0's unique id."""
    from paper_2205_15757_b200 import EUCLIDEAN, Context, Model, ModelGroup
    from paper_2205_15757_b200.dist import assigned_models, share_bytes
    from paper_2205_15757_b200.workload import resnet_group
    N = N or world
    files, digs, sds = resnet_group("resnet50", replicas=N, seed=seed, jitter=5e-3)
    uid = share_bytes(Context.nccl_unique_id() if rank == 0 else None)
    ctx.init_nccl(uid, world, rank)
    ms = [Model.load_cnn(ctx, files[p], digs[p]) for p in assigned_models(world, N, rank)]
    grp = ModelGroup.create_dist(ctx, ms, digs, replica_f(N), EUCLIDEAN, eps, b"group-0",
                                 1, max_batch=B, topk=5)
    return grp, ms, files, digs, sds


def pipeline(grp, ctx, batches, K, D, lag, stream=None):
    """K batches through the pipelined hot path, cold start and full drain:
    ingest D batches ahead of certification (their request-midstate chains
    overlap the forwards), certify each, read its decisions back `lag` steps
    behind, and join every stream at the end. With `stream`, returns the
    device time of the whole region (CUDA events on the context stream)."""
    import torch
    from collections import deque
    nb = len(batches)
    if stream is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
    h0 = time.perf_counter()
    pend = deque(grp.ingest(batches[j % nb]) for j in range(min(D, K)))
    done, sats, labs = deque(), [], []

    def fetch():
        r = grp.fetch_ticket(done.popleft())
        sats.append(r["satisfied"])
        labs.append(r["label"])
    for i in range(K):
        t = pend.popleft()
        grp.certify_ticket(t, sync=False)
        done.append(t)
        if i + D < K:
            pend.append(grp.ingest(batches[(i + D) % nb]))
        while len(done) > lag:
            fetch()
    while done:
        fetch()
    ctx.join()  # every ingest, tail and single-leaf chain of the region
    host_ms = 1e3 * (time.perf_counter() - h0) / K
    ms = None
    if stream is not None:
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    torch.cuda.synchronize()
    return ms, host_ms, sats, labs


def host_hash_ops(batches, threads, slots):
    """hash_ops (messages.cpp:197-202) of `slots` PRE-PREPARE op lists of B
    ImageNet requests each on the host (SHA-NI, one op list per thread)."""
    from paper_2205_15757_b200 import hash_ops_batches
    from paper_2205_15757_b200.credo import lib
    bs = [batches[i % len(batches)] for i in range(slots)]
    hash_ops_batches(bs[:1], b"group-0", [1], threads=1)  # warm
    t = time.perf_counter()
    hash_ops_batches(bs, b"group-0", [1] * slots, threads=threads)
    dt = time.perf_counter() - t
    B = len(bs[0].nonces)
    return {"value": round(slots * B / dt, 1), "unit": "req/s", "threads": threads,
            "sha_ni": bool(lib().cg_host_sha_accelerated()),
            "bytes_per_request": int(bs[0].inputs[0].size * 8 + 200),
            "sample": f"{slots} op lists x {B} requests, {dt:.2f} s"}


def bench_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2205_15757_b200 import Context, lib
    from paper_2205_15757_b200.workload import signed_requests

    torch.cuda.set_device(local_rank)
    ctx = Context(local_rank)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    B = args.batch
    replica = args.mode == "replica"
    if replica:
        grp, models, files, digs, sds = make_dist_group(ctx, B, rank, world,
                                                        N=max(world, args.replicas_dist))
    elif args.workload == "c3":
        grp, models, files, digs, sds = make_hetero_group(ctx, B)
    else:
        grp, models, files, digs, sds = make_group(ctx, B, seed=0)
    # group mode: each rank its own stream; replica mode: one shared stream
    seed_base = 0 if replica else 100 * rank
    jobs = 1 if replica else world  # independent request streams
    L = lib()
    L.cg_model_flops_per_input.restype = __import__("ctypes").c_double
    L.cg_timing_read.argtypes = [__import__("ctypes").c_int,
                                 __import__("ctypes").POINTER(__import__("ctypes").c_double),
                                 __import__("ctypes").POINTER(__import__("ctypes").c_uint64)]
    flops_img = sum(L.cg_model_flops_per_input(m.h) for m in models)  # this rank's replicas

    # Two rotating batches of 154 MB f64 inputs each (> 126 MB L2): plain
    # (pageable) host arrays -- one vector<double> per request, as the
    # reference holds them -- for e2e, device copies for the device-resident
    # value.
    nb = 2
    batches = [signed_requests(B, U, seed=seed_base + i) for i in range(nb)]
    dev_in = [torch.from_numpy(b.inputs).to(f"cuda:{local_rank}") for b in batches]
    from copy import copy
    dev_batches = []
    for b, d in zip(batches, dev_in):
        db = copy(b)
        db.inputs, db.B, db.u = d.data_ptr(), B, U
        dev_batches.append(db)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warmup (also validates: every request must be certified) ----
    for i in range(args.warmup):
        r = grp.certify(batches[i % nb])
    sat = float(np.mean(r["satisfied"]))
    torch.cuda.synchronize()
    if args.profile:  # ncu mode: a few plain steps, nothing else
        for i in range(args.steps):
            grp.certify(dev_batches[i % nb], sync=False)
        torch.cuda.synchronize()
        return {"profile": True, "satisfied": sat}
    D, LAG = args.depth, args.fetch_lag
    if args.trace:  # kineto/CUPTI timeline of the pipelined loop (all streams)
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            pipeline(grp, ctx, dev_batches, args.steps, D, LAG)
        if rank == 0:
            prof.export_chrome_trace(args.trace)
        return {"trace": args.trace}

    # ---- device-resident throughput (value) ----
    # Cold start, full drain: the timed region issues every ingest (framing +
    # request-midstate SHA chains, InferenceEngine::submit's device part, D
    # batches ahead of certification) and every certify of its K batches, and
    # ends when all of their work -- forwards, chains, agreement, trees, the
    # lazily chained single-attestation leaves -- has finished
    # (cg_ctx_join). Decisions are read back LAG steps behind, inside it.
    barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()  # kernels launched inside the timed region only
    with ClockSampler(local_rank) as clk:
        ms, host_ms, sats, labs = pipeline(grp, ctx, dev_batches, args.steps, D, LAG, stream)
    launches = round((ctx.launch_count() - l0) / args.steps)
    if world > 1:  # per-rank device times and SM clocks (stderr; the line reports the max)
        per = torch.zeros(2 * world, dtype=torch.float64, device=f"cuda:{local_rank}")
        per[rank] = ms
        per[world + rank] = clk.summary().get("sm_mhz") or 0.0
        dist.all_reduce(per)
        if rank == 0:
            v = per.tolist()
            print("per-rank ms/step: " + " ".join(f"{x / args.steps:.3f}" for x in v[:world])
                  + " | SM MHz: " + " ".join(f"{x:.0f}" for x in v[world:]), file=sys.stderr)
    ms = max_over_ranks(ms)
    sat_dev = float(np.mean(np.concatenate(sats)))
    label_frac = float(np.mean(np.concatenate(labs) >= 0))
    value = jobs * args.steps * B * sat_dev / (ms / 1e3)

    # ---- fault path: corrupt_result on provider 2 for 30 % of the requests
    # (10 % of the (request, replica) pairs): single-attestation leaves --
    # a 0x53 request midstate per request where provider 2 is in the quorum
    fault = None
    if not replica and args.workload == "c2" and not args.no_fault and not args.quick:
        grp.set_fault(2, 1.0, 0.3)
        # untimed: the stream's first single leaves switch the group to
        # speculative 0x53 midstates (chained at ingest), its steady state
        pipeline(grp, ctx, dev_batches, D + LAG + 2, D, LAG)
        barrier()
        torch.cuda.synchronize()
        fms, _, fsats, _ = pipeline(grp, ctx, dev_batches, args.steps, D, LAG, stream)
        grp.set_fault(2, 0.0, 0.0)
        fms = max_over_ranks(fms)
        fsat = float(np.mean(np.concatenate(fsats)))
        hit = float(np.mean([np.mean(b.request_ids[:, 0] < round(256 * 0.3)) for b in batches]))
        fault = {"value": round(jobs * args.steps * B * fsat / (fms / 1e3), 1), "unit": UNIT,
                 "ms_per_step": round(fms / args.steps, 3),
                 "faulty_pair_fraction": round(hit / 3, 4),
                 "fault": "OffsetExecutor(+1.0) on provider 2 for requests with id[0] < 77 "
                          "(harness.cpp:167-186 corrupt_result)",
                 "satisfied_fraction": fsat,
                 "ratio_to_honest": round((fsat / max(sat_dev, 1e-9)) * (ms / fms), 4)}

    e2e, ms_e2e, host_e2e = None, 0.0, 0.0
    # ---- end to end through the public API: the batch former ----
    # Every step submits B requests (InferenceEngine::submit: structural
    # checks, seen-dedup, packing each request's pageable f64 input into
    # pinned staging on pack threads), the released batch is ingested
    # (framing, H2D of 154 MB, chains), certified, and its decisions + roots
    # are read back LAG steps behind -- all inside the region.
    from collections import deque

    from paper_2205_15757_b200 import InferenceEngine
    if not args.quick:
        e2e, ms_e2e, host_e2e = e2e_leg(args, ctx, grp, batches, B, D, LAG, rank, jobs, stream,
                                        barrier, max_over_ranks)

    h2d = B * U * 8
    d2h = B * (4 + 8 + 1 + 8) + grp.N * 32 + 32 + 8

    # ---- attribution pass: per-kernel-class device time (same pipeline) ----
    import ctypes
    L.cg_timing_enable(1)
    pipeline(grp, ctx, dev_batches, args.steps, D, LAG, stream)
    tg, ng = ctypes.c_double(), ctypes.c_uint64()
    L.cg_timing_read(0, ctypes.byref(tg), ctypes.byref(ng))
    tc, nc = ctypes.c_double(), ctypes.c_uint64()
    L.cg_timing_read(1, ctypes.byref(tc), ctypes.byref(nc))
    # per-launch GEMM times -> efficiency against each layer's own roofline
    # floor max(FLOPs / tensor peak, compulsory bytes / HBM peak)
    spans = (ctypes.c_double * int(ng.value))()
    cnt = ctypes.c_uint64()
    L.cg_timing_spans.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64,
                                  ctypes.POINTER(ctypes.c_uint64)]
    L.cg_timing_spans(0, spans, ng.value, ctypes.byref(cnt))
    floor_eff = None
    if args.workload == "c2" and not replica:
        plan = resnet50_gemm_plan(B, len(models))
        if len(plan) and cnt.value == len(plan) * args.steps:
            pk0, _ = peaks()
            fl = pk0.get("bf16_tflops_sustained", pk0["bf16_tflops"]) * 1e12
            bw = pk0.get("hbm_gbs", 6650.0) * 1e9
            floors = sum(max(f / fl, b / bw) for _, f, b in plan) * args.steps * 1e3
            floor_eff = {"frac": round(floors / sum(spans), 4),
                         "floor_ms_per_step": round(floors / args.steps, 3),
                         "compulsory_bytes_per_step": int(sum(b for _, _, b in plan))}
    breakdown = {}
    for cls, name in ((2, "agree_trees_ms"), (3, "aux_ms"), (4, "nccl_ms")):
        t, n = ctypes.c_double(), ctypes.c_uint64()
        L.cg_timing_read(cls, ctypes.byref(t), ctypes.byref(n))
        breakdown[name] = round(t.value / args.steps, 3)
    L.cg_timing_enable(0)
    gemm_ms_step = tg.value / args.steps
    chain_ms_step = tc.value / args.steps
    pk, pk_src = peaks()
    flops_step = B * flops_img
    achieved = flops_step / (gemm_ms_step / 1e3) / 1e12
    peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    traffic, traffic_src = None, None
    if args.workload == "c2" and not replica:
        try:  # DRAM bytes of one step's GEMM launches, from the committed ncu capture
            with open(os.path.join(ROOT, "profiles", "r02_gemm_step_traffic.json")) as f:
                tj = json.load(f)
            traffic, traffic_src = tj["traffic_bytes_per_step"], tj["source"]
        except Exception:
            pass
    roofline = {"bound": "tensor", "kernel": "conv_gemm (tcgen05 implicit-GEMM, all convs+fc)",
                "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_unit": "DRAM bytes per step (all conv_gemm launches)",
                "traffic_source": traffic_src,
                "peak_source": f"{pk_src} bf16_tflops_sustained",
                "algorithmic_flops_per_step": flops_step,
                "gemm_ms_per_step": round(gemm_ms_step, 3),
                "gemm_launches_per_step": int(ng.value) // args.steps,
                "share_of_step": round(gemm_ms_step / (ms / args.steps), 3),
                "sha_chain_ms_per_step_overlapped": round(chain_ms_step, 3),
                "other_ms_per_step": breakdown,
                "per_layer_floor": floor_eff}

    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(ms / args.steps, 3), "host_ms_per_step": round(host_ms, 3),
           "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic (random-init jittered ResNet-50 replicas, U(-1,1) f64 "
                   "requests, Ed25519-signed)",
           "config": {**c2_config(B, world),
                      "l2": "inputs larger than L2: 2 rotating 154 MB f64 batches",
                      "arith": "bf16 forward / f64 agreement / u32 SHA-256",
                      "satisfied_fraction": sat_dev,
                      "pipeline": f"cold start + full drain inside the region: ingest {D} "
                                  f"batches ahead (request-midstate SHA chains overlap the "
                                  f"forwards), decisions read back {LAG} steps behind"},
           "e2e": None if e2e is None else {"value": round(e2e, 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h, "ms_per_step": round(ms_e2e / args.steps, 3),
                   "host_s": round(host_e2e, 3), "steps": max(args.steps, 60),
                   "path": "InferenceEngine.submit of B requests per step (structural checks, "
                           "dedup, pack of pageable per-request f64 inputs into pinned staging "
                           f"on {args.pack_threads} threads) -> ingest (154 MB H2D) -> certify "
                           "-> decisions + roots read back, all in the region"},
           "fault_path": fault,
           "gpu_launches": int(launches),
           "roofline": roofline,
           "clocks": clk.summary()}
    if rank == 0 and not replica and args.workload == "c2" and not args.quick:
        out["host_hash_ops"] = host_hash_ops(batches, os.cpu_count() or 1, 16)
    if args.workload == "c3":
        from paper_2205_15757_b200.workload import HETERO_GROUP
        out["metric"] = METRIC.replace("(ResNet-50 group)", "(heterogeneous group)")
        out["config"].update(
            workload="C3: heterogeneous 4-replica group (ResNet-50, ResNet-101, VGG-16, "
                     f"MobileNetV2), f=1, batch {B}, 224x224 (BASELINE.json configs[2])",
            model="+".join(HETERO_GROUP), replicas=4, f=1, epsilon=C3_EPS,
            labels_agreed_fraction=label_frac)
    if replica:
        out["scaling"] = "strong"
        out["config"].update(
            workload=f"{grp.N}-replica ResNet-50 group, {grp.N // world} replica(s) per GPU, "
                     f"f={replica_f(grp.N)}, batch {B}, 224x224; outputs + R roots "
                     "all-gathered over NCCL",
            replicas=grp.N, f=replica_f(grp.N), global_batch=B,
            parallelism=f"replica-parallel x{world} (rank = provider chunk, assigned_models)")
    if world == 1 and not args.no_cpu_baseline and not args.quick:  # timed at N=1 only
        archs = [m.arch for m in models] if args.workload == "c3" else ["resnet50"] * 3
        out["cpu_baseline"] = cpu_baseline(archs, digs, sds, batches[0], args,
                                           grp.default_eps)
    return out


def e2e_leg(args, ctx, grp, batches, B, D, LAG, rank, jobs, stream, barrier, max_over_ranks):
    """Cold start and full drain like the value leg, over max(K, 60) steps
    (the region starts with no batch in flight and ends with the last
    batch's 35 ms request-midstate chain, so a short region would mostly
    measure that latency). Batches are certified 2 steps after submission:
    the forwards do not wait for the chains (only the certification tail
    does), so deeper read-ahead only delays the first forward."""
    import torch
    from collections import deque

    from paper_2205_15757_b200 import InferenceEngine
    from paper_2205_15757_b200.workload import signed_requests
    nb = len(batches)
    K = max(args.steps, 60)
    D = min(D, 2)
    eng = InferenceEngine(ctx, B, 10**12, pack_threads=args.pack_threads)
    eng.load_group(grp)
    # K distinct signed batches (the engine's seen-dedup absorbs repeats);
    # their inputs share the two 154 MB arrays' rows, the pack still copies
    # every request's 1.2 MB into pinned staging
    e2e_batches = [signed_requests(B, U, seed=10_000 + 100 * rank + i,
                                   inputs=batches[i % nb].inputs) for i in range(K)]
    prepared = [eng.prepare(b, b"group-0") for b in e2e_batches]
    # untimed warm-up with other requests: the engine's pinned staging and
    # every ingest slot's device input buffer get allocated here
    warm = [eng.prepare(signed_requests(B, U, seed=20_000 + 100 * rank + i,
                                        inputs=batches[i % nb].inputs), b"group-0")
            for i in range(min(grp.ring, D + LAG + 4))]
    wq = deque()
    for i, w in enumerate(warm):
        eng.submit_prepared(w, now_us=i)
        for gq, _, t, Bt in eng.ready():
            gq.certify_ticket(t, sync=False, B=Bt)
            wq.append(t)
        while len(wq) > LAG:
            grp.fetch_ticket(wq.popleft())
    while wq:
        grp.fetch_ticket(wq.popleft())
    ctx.join()
    barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    h2 = time.perf_counter()
    certified = 0
    ready_q, inflight = deque(), deque()

    def certify_oldest():
        grp_, _, t, Bt = ready_q.popleft()
        grp_.certify_ticket(t, sync=False, B=Bt)
        inflight.append(t)

    def fetch_oldest():
        return int(np.sum(grp.fetch_ticket(inflight.popleft())["satisfied"]))
    for i in range(K):
        eng.submit_prepared(prepared[i], now_us=i)  # one full batch of B per step
        ready_q.extend(eng.ready())
        while len(ready_q) > D:
            certify_oldest()
        while len(inflight) > LAG:
            certified += fetch_oldest()
    while ready_q:
        certify_oldest()
    while inflight:
        certified += fetch_oldest()
    ctx.join()
    e3.record(stream)
    torch.cuda.synchronize()
    host_e2e = time.perf_counter() - h2
    ms_e2e = max_over_ranks(e2.elapsed_time(e3))
    e2e = jobs * certified / (ms_e2e / 1e3)
    eng.free()
    return e2e, ms_e2e * args.steps / K, host_e2e  # ms scaled to per-step below



# ------------------------------------------------------------ CPU baseline
def cpu_models(archs, sds):
    """The replicas as torchvision CPU modules (loaded once, like the
    reference's InferenceEngine::load_group, outside any timed region)."""
    from oracle import cnn_oracle
    return [cnn_oracle.build(arch, sd) for arch, sd in zip(archs, sds)]


def cpu_path(models, encs, inputs, digs, threads, R, eps=0.1):
    """The reference's CPU path for a sample: torchvision fp32 forward per
    replica (restatement: the reference has no CNN), then the compiled
    reference's select_quorum, ensemble_label, result leaves, R trees,
    manifest and A tree (oracle/_ref ref_certify_batch). Returns (result,
    forward seconds, agreement + digest seconds)."""
    import torch

    from oracle import cnn_oracle
    torch.set_num_threads(threads)
    t0 = time.perf_counter()
    outs = []
    for m in models:
        outs.append(cnn_oracle.softmax_f64(cnn_oracle.logits(m, inputs)))
    outs = np.stack(outs)
    t1 = time.perf_counter()
    h = R.batch_new(encs, 1)
    r = R.certify_batch(h, len(models), 1, 0, eps, outs, 1, digs, threads=threads)
    R.batch_free(h)
    return r, t1 - t0, time.perf_counter() - t1


def cpu_digest_seconds(backend: str, threads: int, S: int, N: int = 3) -> float:
    """Agreement + digest part of the reference's CPU path (select_quorum,
    labels, result leaves, R trees, manifest, A tree) for S ImageNet-shaped
    requests with the given SHA-256 backend. Runs in its own process (the two
    reference builds export the same libsodium symbols)."""
    from oracle.oracle import Reference
    from paper_2205_15757_b200.workload import encode_request, signed_requests
    batch = signed_requests(S, U, seed=0)
    encs = [encode_request(batch, k) for k in range(S)]
    rng = np.random.default_rng(1)
    base = rng.dirichlet(np.ones(1000), S)
    outs = np.stack([base + rng.uniform(-1e-6, 1e-6, base.shape) for _ in range(N)])
    digs = [bytes([p]) * 32 for p in range(N)]
    R = Reference(backend)
    h = R.batch_new(encs, 1)
    t = time.perf_counter()
    R.certify_batch(h, N, 1, 0, 0.1, outs, 1, digs, threads=threads)
    dt = time.perf_counter() - t
    R.batch_free(h)
    return dt


def _digest_seconds_subprocess(backend, threads, S):
    code = (f"import sys; sys.path.insert(0, {ROOT!r}); import bench; "
            f"print(bench.cpu_digest_seconds({backend!r}, {threads}, {S}))")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600)
    return float(out.stdout.strip().splitlines()[-1])


def cpu_baseline(archs, digs, sds, batch, args, eps=0.1):
    from oracle.oracle import Reference
    from paper_2205_15757_b200.workload import encode_request
    threads = os.cpu_count() or 1
    S = max(1, args.cpu_sample)
    # the sample cycles through the batch's requests when S > batch size
    nb = len(batch.inputs)
    idx = [k % nb for k in range(S)]
    encs = [encode_request(batch, k) for k in idx]
    kind = "reference" if Reference.available() else "port"
    if kind != "reference":
        return {"value": None, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": "oracle/_ref not built on this box"}
    R = Reference()
    models = cpu_models(archs, sds)
    cpu_path(models, encs[:2], batch.inputs[:2], digs, threads, R, eps)  # warm
    _, t_fwd, t_dig = cpu_path(models, encs, np.take(batch.inputs, idx, axis=0), digs,
                               threads, R, eps)
    dt = t_fwd + t_dig
    out = {"value": round(S / dt, 3), "unit": UNIT, "cores": threads, "kind": kind,
           "sample": f"{S} requests x {len(archs)} replicas ({'+'.join(sorted(set(archs)))}): "
                     f"torchvision fp32 forward (restated; "
                     f"the reference has no CNN) + compiled reference select_quorum/"
                     f"ensemble_label/result leaves/R+A trees, {dt:.1f} s "
                     f"(forward {t_fwd:.1f} s, agreement + digests {t_dig:.2f} s), "
                     "SHA-256 via OpenSSL (SHA-NI)"}
    # the same with the SHA-256 the reference ships (libsodium), and on one
    # core (a smaller sample, scaled)
    try:
        Sd = min(S, 64)
        t_sod = _digest_seconds_subprocess("libsodium", threads, Sd) * S / Sd
        S1 = 4
        _, f1, _ = cpu_path(models, encs[:S1], np.take(batch.inputs, idx[:S1], axis=0), digs, 1,
                            R, eps)
        d1 = _digest_seconds_subprocess("openssl", 1, 16) / 16
        d1s = _digest_seconds_subprocess("libsodium", 1, 8) / 8
        out["backends"] = {
            "openssl_all_cores": round(S / dt, 3),
            "libsodium_all_cores": round(S / (t_fwd + t_sod), 3),
            "openssl_1_core": round(1.0 / (f1 / S1 + d1), 3),
            "libsodium_1_core": round(1.0 / (f1 / S1 + d1s), 3),
            "digest_only_req_per_s": {"openssl_all_cores": round(S / t_dig, 1),
                                      "libsodium_all_cores": round(S / t_sod, 1),
                                      "openssl_1_core": round(1 / d1, 1),
                                      "libsodium_1_core": round(1 / d1s, 1)}}
    except Exception as e:  # noqa: BLE001
        out["backends"] = {"error": str(e)[:200]}
    return out


# ------------------------------------------------------------ C4 update
def bench_c4(args, rank, world, local_rank):
    """C4 (BASELINE.json configs[3]): an N-replica ResNet-50 group, f =
    (N-1)//3, batch 512, with a concurrent model-version update mid-stream.
    One GPU: the N (default 8) replicas time-sliced on it; N GPUs: one model
    owner per GPU (rank = provider, outputs + R roots all-gathered over NCCL).

    Inside the timed region:
      * v1 serves alone;
      * at step K//3 a background thread loads v2 -- every replica file's
        SHA-256 check (load_group, engine.cpp:79), parse + BN fold, upload --
        and creates its group while v1 keeps certifying (v2 = a new jitter
        salt, harness.cpp:601-602);
      * once v2 is resident (the same step on every rank) each batch is
        ingested and certified under BOTH live versions (engine.cpp:196-206);
      * v1 retires at step 2K//3 (or D+1 steps after v2 went live, if later);
    a request counts once if satisfied under at least one version (the
    host-side version fold, state.cpp:23-45). Every batch's decisions are
    read back inside the region; the region ends when all work is drained."""
    import threading

    import torch
    import torch.distributed as dist
    from collections import deque

    from paper_2205_15757_b200 import EUCLIDEAN, Context, Model, ModelGroup
    from paper_2205_15757_b200.dist import assigned_models, share_bytes
    from paper_2205_15757_b200.workload import resnet_group, signed_requests
    torch.cuda.set_device(local_rank)
    ctx = Context(local_rank)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    # N replicas (default 8): on N GPUs one per GPU; on fewer GPUs that
    # divide N, assigned_models chunks of N / world per rank; on one GPU
    # all N time-sliced
    B = args.batch
    N = args.replicas if args.replicas % max(world, 1) == 0 and args.replicas >= world else world
    f = (N - 1) // 3
    eps = 0.1
    gloo = None
    if world > 1:
        uid = share_bytes(Context.nccl_unique_id() if rank == 0 else None)
        ctx.init_nccl(uid, world, rank)
        gloo = dist.new_group(backend="gloo")
    files = {}
    for version, salt in ((1, 0), (2, 1000)):  # model files on disk: setup, untimed
        fl, dg, _ = resnet_group("resnet50", replicas=N, seed=0, jitter=5e-3, salt=salt)
        files[version] = (fl, dg)

    def load(version):
        fl, dg = files[version]
        if world > 1:
            ms = [Model.load_cnn(ctx, fl[p], dg[p]) for p in assigned_models(world, N, rank)]
            g = ModelGroup.create_dist(ctx, ms, dg, f, EUCLIDEAN, eps, b"group-0", version,
                                       max_batch=B, topk=5)
        else:
            ms = [Model.load_cnn(ctx, x, d) for x, d in zip(fl, dg)]
            g = ModelGroup(ctx, ms, f, EUCLIDEAN, eps, b"group-0", version, max_batch=B, topk=5)
        return g, ms

    t_load0 = time.perf_counter()
    g1, ms1 = load(1)
    v1_load_s = time.perf_counter() - t_load0
    nb = 2
    batches = [signed_requests(B, U, seed=7 + i) for i in range(nb)]
    dev = []
    for b in batches:
        d = torch.from_numpy(b.inputs).to(f"cuda:{local_rank}")
        db = copy.copy(b)
        db.inputs, db.B, db.u = d.data_ptr(), B, U
        db._keep = d
        dev.append(db)
    for i in range(args.warmup):
        g1.certify(dev[i % nb])
    torch.cuda.synchronize()
    K, D, LAG = args.steps, min(args.depth, 6), min(args.fetch_lag, 6)
    groups = {1: g1}
    loaded, loader = {}, None
    v2_live_at, v1_retired_at = None, None

    def agreed(flag):  # the same decision on every rank (gloo: no GPU sync)
        if world == 1:
            return flag
        t = torch.tensor([1 if flag else 0])
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=gloo)
        return bool(t.item())

    tickets = {}  # batch -> [(version, ticket)]
    done, sat_by_batch = deque(), {}

    def ingest(j, live):
        tickets[j] = [(v, groups[v].ingest(dev[j % nb])) for v in live]

    def fetch_one():
        j, v, t = done.popleft()
        s_ = groups[v].fetch_ticket(t)["satisfied"].astype(bool)
        sat_by_batch[j] = s_ if j not in sat_by_batch else (sat_by_batch[j] | s_)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    certs = 0
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        h0 = time.perf_counter()
        live = [1]
        for j in range(min(D, K)):
            ingest(j, live)
        for i in range(K):
            if i == K // 3:
                def bg():
                    t = time.perf_counter()
                    loaded["g"] = load(2)
                    loaded["s"] = time.perf_counter() - t
                loader = threading.Thread(target=bg)
                loader.start()
            if v2_live_at is None and i > K // 3 and agreed("g" in loaded):
                loader.join()
                groups[2] = loaded["g"][0]
                v2_live_at = i
                live = [1, 2]
            if (v2_live_at is not None and v1_retired_at is None
                    and i >= max(2 * K // 3, v2_live_at + D + 1)):
                v1_retired_at = i
                live = [2]
            for v, t in tickets.pop(i):
                groups[v].certify_ticket(t, sync=False)
                done.append((i, v, t))
                certs += 1
            if i + D < K:
                ingest(i + D, live)
            while len(done) > LAG * len(live):
                fetch_one()
        while done:
            fetch_one()
        ctx.join()
        e1.record(stream)
        torch.cuda.synchronize()
        host_s = time.perf_counter() - h0
    if loader is not None and loader.is_alive():
        loader.join()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local_rank}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    certified = int(sum(int(np.sum(s_)) for s_ in sat_by_batch.values()))
    value = certified / (ms / 1e3)
    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
           "steps": K, "warmup": args.warmup, "ms_per_step": round(ms / K, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic (random-init jittered ResNet-50 replicas, v2 = new jitter salt)",
           "config": {"workload": f"C4: {N}-replica ResNet-50 group, f={f}, batch {B}, "
                                  f"{f'{N // world} replica(s) per GPU over NCCL' if world > 1 else 'time-sliced on 1 GPU'}"
                                  ", v1 -> v2 update mid-stream, v2 loaded inside the timed "
                                  "region (BASELINE.json configs[3])",
                      "model": "resnet50", "replicas": N, "f": f, "global_batch": B,
                      "v2_load_started_step": K // 3, "v2_live_step": v2_live_at,
                      "v1_retired_step": v1_retired_at,
                      "v2_load_s": round(loaded.get("s", float("nan")), 2),
                      "v1_load_s_untimed": round(v1_load_s, 2),
                      "certifications_per_request": round(certs / K, 3),
                      "certified_requests": certified, "requests": K * B,
                      "host_s": round(host_s, 2),
                      "parallelism": f"replica-parallel x{world}" if world > 1 else "1 GPU",
                      "l2": f"inputs larger than L2: 2 rotating {B * U * 8 >> 20} MB f64 batches"},
           "clocks": clk.summary()}
    for g in groups.values():
        g.free()
    return out


# ------------------------------------------------------------- C1
def bench_c1(args, rank, world, local_rank):
    """C1 (BASELINE.json configs[0]): the reference's default group at SURVEY
    §8(d)'s shape -- three generate_group LinearToyModels 3072 -> 10 with
    softmax (the compiled reference's own model files, tests/golden/
    c1_full.npz), f=1, batch 64, euclidean eps 0.05 -- through the same
    pipelined path as C2: fp64 LinearToyModel kernel (bit-exact), softmax /
    top-k, agreement + label, result leaves (~26 KB hashed per request), R
    and A trees. 100 rotating batches (157 MB of inputs > L2)."""
    import torch

    from paper_2205_15757_b200 import EUCLIDEAN, Context, Model, ModelGroup
    from paper_2205_15757_b200.workload import signed_requests
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    g = np.load(os.path.join(ROOT, "tests", "golden", "c1_full.npz"))
    torch.cuda.set_device(local_rank)
    ctx = Context(local_rank)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    N, B, u = int(g["N"]), int(g["B"]), int(g["u"])
    models = [Model.load_linear(ctx, g["files"][p].tobytes(), g["digests"][p].tobytes())
              for p in range(N)]
    grp = ModelGroup(ctx, models, 1, EUCLIDEAN, float(g["eps"]), g["gid"].tobytes(), 1,
                     max_batch=B, topk=5)
    nb = max(100, args.steps)  # distinct batches: the batch former dedups repeats
    batches = [signed_requests(B, u, seed=1000 + rank * nb + i) for i in range(nb)]
    dev = []
    for b in batches:
        d = torch.from_numpy(b.inputs).to(f"cuda:{local_rank}")
        db = copy.copy(b)
        db.inputs, db.B, db.u = d.data_ptr(), B, u
        db._keep = d
        dev.append(db)
    for i in range(args.warmup):
        grp.certify(batches[i % nb])
    torch.cuda.synchronize()
    D, LAG = args.depth, args.fetch_lag
    l0 = ctx.launch_count()
    with ClockSampler(local_rank) as clk:
        ms, host_ms, sats, _ = pipeline(grp, ctx, dev, args.steps, D, LAG, stream)
    launches = round((ctx.launch_count() - l0) / args.steps)
    sat = float(np.mean(np.concatenate(sats)))
    value = world * args.steps * B * sat / (ms / 1e3)
    # e2e: the batch former from pageable host inputs
    from paper_2205_15757_b200 import InferenceEngine
    eng = InferenceEngine(ctx, B, 10**12, pack_threads=2)
    eng.load_group(grp)
    prepared = [eng.prepare(b, g["gid"].tobytes()) for b in batches]
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    from collections import deque
    ready_q, inflight, certified = deque(), deque(), 0
    for i in range(args.steps):
        eng.submit_prepared(prepared[i % nb], now_us=i)  # nb = 100 distinct batches
        ready_q.extend(eng.ready())
        while len(ready_q) > D:
            gq, _, t, Bt = ready_q.popleft()
            gq.certify_ticket(t, sync=False, B=Bt)
            inflight.append(t)
        while len(inflight) > LAG:
            certified += int(np.sum(grp.fetch_ticket(inflight.popleft())["satisfied"]))
    while ready_q:
        gq, _, t, Bt = ready_q.popleft()
        gq.certify_ticket(t, sync=False, B=Bt)
        inflight.append(t)
    while inflight:
        certified += int(np.sum(grp.fetch_ticket(inflight.popleft())["satisfied"]))
    ctx.join()
    e3.record(stream)
    torch.cuda.synchronize()
    e2e = world * certified / (e2.elapsed_time(e3) / 1e3)
    eng.free()
    # digest work per request: the shared request midstate (386 blocks) + N
    # result-leaf tails + the A/R tree nodes, in SHA-256 blocks of 64 B
    req_len = len(bytes(g["reqs"].tobytes())) // B
    blocks = (req_len + 2) // 64 + N * 4 + 2 * N + 4
    hashed = blocks * 64 * B * args.steps * sat
    pk, pk_src = peaks()
    out = {"metric": METRIC.replace("(ResNet-50 group)", "(C1 LinearToyModel group)"),
           "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
           "host_ms_per_step": round(host_ms, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64 (LinearToyModel, bit-exact)",
           "data": "the compiled reference's generate_group models (seed 7, softmax); "
                   "synthetic signed U(-1,1) requests",
           "config": {"workload": "C1: 3 x LinearToyModel 3072->10 softmax, f=1, batch 64, "
                                  "eps 0.05 (BASELINE.json configs[0], SURVEY §8(d))",
                      "replicas": N, "f": 1, "batch_per_gpu": B, "satisfied_fraction": sat,
                      "l2": "100 rotating batches, 157 MB of inputs > L2",
                      "pipeline": f"cold start + full drain, ingest {D} ahead, read back "
                                  f"{LAG} behind"},
           "e2e": {"value": round(e2e, 1), "unit": UNIT, "h2d_bytes_per_step": B * u * 8,
                   "d2h_bytes_per_step": B * 21 + N * 32 + 40,
                   "path": "InferenceEngine.submit -> ingest -> certify -> read back"},
           "gpu_launches": int(launches),
           "roofline": {"bound": "latency (SHA-256 chains, one thread per chain)",
                        "achieved": round(hashed / (ms / 1e3) / 1e9, 2),
                        "peak": pk.get("hbm_gbs", 6650.0), "unit": "GB/s",
                        "frac": round(hashed / (ms / 1e3) / 1e9 / pk.get("hbm_gbs", 6650.0), 5),
                        "traffic": None,
                        "note": "bytes hashed per second against HBM bandwidth: C1 is bound "
                                "by the per-request SHA chain latency and launch overheads, "
                                "not by a roofline"},
           "clocks": clk.summary()}
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = c1_cpu_baseline(g, batches[0], args)
    grp.free()
    for m in models:
        m.free()
    return out


def c1_cpu_baseline(g, batch, args):
    """The compiled reference's C1 path on the host cores: LinearToyModel::run
    per replica (ref_linear_run) + select_quorum / ensemble_label / leaves /
    trees (ref_certify_batch); all cores, a bounded sample."""
    from oracle.oracle import Reference
    from paper_2205_15757_b200.workload import encode_request
    if not Reference.available():
        return {"value": None, "kind": "port", "sample": "oracle/_ref not built"}
    R = Reference()
    threads = os.cpu_count() or 1
    N, v = int(g["N"]), int(g["v"])
    gid = g["gid"].tobytes()
    encs = [encode_request(batch, k, gid) for k in range(len(batch.nonces))]
    digs = [g["digests"][p].tobytes() for p in range(N)]
    h = R.batch_new(encs, 1)
    reps = 0
    t = time.perf_counter()
    while time.perf_counter() - t < 5.0:
        outs = np.stack([R.linear_run(g["files"][p].tobytes(), batch.inputs, v) for p in range(N)])
        R.certify_batch(h, N, 1, 0, float(g["eps"]), outs, 1, digs, threads=threads)
        reps += 1
    dt = time.perf_counter() - t
    R.batch_free(h)
    return {"value": round(reps * len(encs) / dt, 1), "unit": UNIT, "cores": threads,
            "kind": "reference",
            "sample": f"{reps} batches x {len(encs)} requests, LinearToyModel::run x {N} "
                      f"(single thread) + certify_batch ({threads} threads), {dt:.1f} s"}


# ------------------------------------------------------------- C5 sweep
def bench_c5(args, local_rank):
    """C5 (BASELINE.json configs[4]): agreement + compact label digests over
    R precomputed per-replica results resident in HBM (cg_agree_device, one
    launch per step). One JSON line per (R, n, v)."""
    import torch

    from paper_2205_15757_b200 import Context
    from paper_2205_15757_b200.workload import signed_requests  # noqa: F401  (import check)
    torch.cuda.set_device(local_rank)
    dev = torch.device(f"cuda:{local_rank}")
    ctx = Context(local_rank)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    pk, pk_src = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    lines = []
    for spec in args.c5.split(","):
        R, n, v = (int(float(x)) for x in spec.split("x"))
        f = 1 if n <= 4 else 2
        outs = torch.empty(n * R * v, dtype=torch.float64, device=dev)
        ids = torch.empty(R * 32, dtype=torch.uint8, device=dev)
        ctx.synth_outputs(0xC5, R, n, v, 0.05, 0.1, outs.data_ptr(), ids.data_ptr())
        eps = torch.full((R,), 0.05, dtype=torch.float64, device=dev)
        sel = torch.empty(R, dtype=torch.int32, device=dev)
        diam = torch.empty(R, dtype=torch.float64, device=dev)
        sat = torch.empty(R, dtype=torch.uint8, device=dev)
        st = torch.empty(R, dtype=torch.int8, device=dev)
        lab = torch.empty(R, dtype=torch.int64, device=dev)
        dig = torch.empty(R * 32, dtype=torch.uint8, device=dev)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2

        def step():
            ctx.agree_device(outs.data_ptr(), R * v, v, eps.data_ptr(), R, n, f, v, 0,
                             sel.data_ptr(), diam.data_ptr(), sat.data_ptr(), st.data_ptr(),
                             lab.data_ptr(), ids.data_ptr(), 1, dig.data_ptr())
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        l0 = ctx.launch_count()
        ms = 0.0
        with ClockSampler(local_rank) as clk:
            for _ in range(args.steps):
                flush.zero_()  # L2 flush between timed launches (outside the events)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
                torch.cuda.synchronize()
                ms += e0.elapsed_time(e1)
        launches = (ctx.launch_count() - l0) // args.steps
        per = ms / args.steps
        bytes_req = n * v * 8 + 8 + 32 + (4 + 8 + 1 + 1 + 8 + 32)
        achieved = bytes_req * R / (per / 1e3) / 1e9
        satf = float(sat.float().mean().item())
        lines.append({
            "metric": "C5 agreement + label-digest results/s (device-resident)",
            "value": round(R / (per / 1e3), 1), "unit": "req/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(per, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 agreement / u32 SHA-256", "data": "synthetic (device generator)",
            "config": {"workload": f"C5 R={R} n={n} f={f} v={v} euclidean eps=0.05",
                       "l2": "256 MB buffer written between timed launches",
                       "satisfied_fraction": round(satf, 4)},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": "agree_rows_kernel" if R >= 4096 else
                         "select_quorum_kernel + label_digest_kernel",
                         "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "traffic": None,
                         "peak_source": f"{pk_src} hbm_gbs",
                         "algorithmic_bytes_per_request": bytes_req},
            "clocks": clk.summary()})
        del outs, ids, flush
        torch.cuda.empty_cache()
    return lines


def c2_config(B, world):
    """The C2 workload keys both arms report (BASELINE.json configs[1])."""
    return {"workload": "C2: 3-replica ResNet-50 group, f=1, batch 128, "
                        "224x224 (BASELINE.json configs[1])",
            "model": "resnet50", "replicas": 3, "f": 1, "global_batch": B * world,
            "batch_per_gpu": B, "epsilon": 0.1, "distance": "euclidean",
            "seq_len": None, "parallelism": f"group-per-GPU x{world}"}


def bench_reference(args, rank, world):
    """--impl reference: the reference's CPU path on the host cores."""
    if rank != 0:
        return None
    from oracle.oracle import Reference
    from paper_2205_15757_b200.workload import encode_request, resnet_state_dicts, signed_requests
    import hashlib
    from paper_2205_15757_b200.workload import cnn_model_file
    threads = os.cpu_count() or 1
    sds = resnet_state_dicts("resnet50", 3, seed=0, jitter=5e-3)
    digs = [hashlib.sha256(cnn_model_file("resnet50", sd, U, 1000, True)).digest() for sd in sds]
    # K steps of a bounded sample each, so the whole run stays within a few
    # minutes whatever --steps is: about 2 x cpu_sample requests in total
    K = max(1, args.steps)
    S = max(4, (2 * args.cpu_sample) // K)
    batch = signed_requests(S, U, seed=0)
    encs = [encode_request(batch, k) for k in range(S)]
    if not Reference.available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libcredo_ref.so not built"}
    R = Reference()
    models = cpu_models(["resnet50"] * 3, sds)
    cpu_path(models, encs[:2], batch.inputs[:2], digs, threads, R)  # one small warm-up
    t = time.perf_counter()
    for _ in range(K):
        cpu_path(models, encs, batch.inputs, digs, threads, R)
    dt = time.perf_counter() - t
    v = K * S / dt
    return {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT,
            "n_gpus": world, "steps": K, "warmup": 1,
            "ms_per_step": round(1e3 * dt / K, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 forward / f64 agreement",
            "data": "synthetic", "config": {**c2_config(args.batch, world),
                                            "sample_per_step": S},
            "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": threads,
                             "kind": "reference",
                             "sample": f"{S} requests per step, torchvision fp32 forward "
                                       "(restated) + compiled reference agreement/digests"},
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


_JSON_OUT = None


def emit(obj):
    f = _JSON_OUT or sys.stdout
    f.write(json.dumps(obj) + "\n")
    f.flush()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=None,
                    help="requests per batch (default 128; 512 for --workload c4)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=256,
                    help="requests in the bounded CPU-baseline sample (~10-30 s of CPU work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--depth", type=int, default=12,
                    help="batches ingested ahead of certification (ring holds 24)")
    ap.add_argument("--replicas-dist", type=int, default=0,
                    help="--mode replica: group size (default = number of GPUs; a multiple "
                         "of it gives several replicas per rank)")
    ap.add_argument("--fetch-lag", type=int, default=8,
                    help="steps between certifying a batch and reading its results back")
    ap.add_argument("--pack-threads", type=int, default=8,
                    help="host threads packing request inputs into pinned staging (e2e)")
    ap.add_argument("--no-fault", action="store_true",
                    help="skip the corrupt_result fault-path measurement")
    ap.add_argument("--quick", action="store_true",
                    help="A/B mode: value + GEMM attribution only (no e2e, fault, "
                         "hash_ops or CPU baseline legs)")
    ap.add_argument("--mode", default="group", choices=["group", "replica"],
                    help="group: a whole 3-replica group per GPU (weak scaling); "
                         "replica: one replica per GPU, NCCL all-gather (N>1)")
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="c2: the headline certified-request pipeline (3x ResNet-50); "
                         "c3: the heterogeneous 4-replica group; c5: agreement + "
                         "label-digest sweep (one line per --c5 spec)")
    ap.add_argument("--replicas", type=int, default=8,
                    help="--workload c4: group size on one GPU (N GPUs: N replicas)")
    ap.add_argument("--c5", default="1e6x8x1000,1e6x4x1000,1e6x8x10,1e5x8x1000,1e4x8x1000,"
                                    "1e3x8x1000",
                    help="comma list of RxNxV for --workload c5")
    ap.add_argument("--trace", default=None,
                    help="write a CUPTI timeline (chrome trace JSON) of --steps "
                         "pipelined steps instead of timing")
    ap.add_argument("--profile", action="store_true",
                    help="ncu mode: warmup + --steps plain steps, no report")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.batch is None:
        args.batch = {"c4": 512, "c1": 64}.get(args.workload, 128)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.mode == "replica" and world < 2:
        ap.error("--mode replica needs torchrun with >= 2 ranks")
    # Native libraries (NCCL's version banner) may print to fd 1; route it to
    # stderr while working so stdout carries exactly the JSON line(s).
    json_fd = os.dup(1)
    sys.stdout.flush()
    os.dup2(2, 1)
    global _JSON_OUT
    _JSON_OUT = os.fdopen(json_fd, "w")
    if world > 1:
        import torch.distributed as dist
        if args.impl == "reference":
            if rank != 0:
                return
        else:
            import torch
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    if args.impl == "reference":
        out = bench_reference(args, rank, world)
    elif args.workload == "c4":
        out = bench_c4(args, rank, world, local_rank)
    elif args.workload == "c1":
        out = bench_c1(args, rank, world, local_rank)
    elif args.workload == "c5":
        for line in bench_c5(args, local_rank):
            emit(line)
        return
    else:
        out = bench_gpu(args, rank, world, local_rank)
    if rank == 0 and out is not None:
        emit(out)
    if world > 1 and args.impl != "reference":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
