#!/usr/bin/env python
"""Routed requests/sec of the B200 scheduling hot path (BASELINE.json metric).

Workload (default): BASELINE config 4, the bursty multi-LLM trace -- L ~ lognormal(2048, cv 1)
in [64, 32768] tokens, 512 shared system prefixes, 10% unprofiled requests -- on 256 replicas
(8 models x 32), 16-token blocks, kv 100k / L2 200k tokens per replica.  The trace arrives in
bursts of 125,000 requests per GPU; 8 bursts = the config's 1M requests.  `--workload
long_context` is config 3 (32,768-token prompts, 64 replicas, kv 141k: capacity-bound).

One step = one burst through the whole hot path on a cluster whose state carries over
(paper_2604_25899_b200/steady.py): release of burst k-2 (its placements complete) ->
node table = background + burst k-1's placements -> registry updates -> K2 staged matrix ->
K3 sequential-commit route -> K4/K5 admission (evict_for_space, promoted L2/L3 spans erased in
engine order, insert_chain).  K1 (chain hashing) of burst k+1 runs on a second stream during
step k; every step still hashes its own burst inside the timed region.  Every step routes a
DISTINCT burst; L1 starts near full (warm fill) so admissions evict.

  value  : routed requests/s with the bursts resident in HBM (CUDA events, max over ranks)
  e2e    : the same steps through the public API from pinned HOST buffers: every burst's
           tokens + metadata copied host->device and decisions/admissions/lookups copied back
           inside the timed region
  --impl reference : the unmodified reference (oracle/_ref) through the identical burst
           sequence (same seeds, cluster, warm state), each burst a bounded prefix sample,
           node_view staged values over all host threads
  --check K : K full-size bursts on the GPU and through the reference; compares every
           decision, admission, lookup, staged value and, at the end, every tier

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--check K]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# FNV-1a arithmetic ceiling of one B200 (tools/k1/fnv_core.cu, profiles/r01_fnv_core.txt):
# 513 Gtok/s with register-resident tokens = 4.11 TB/s of token bytes -- K1 is INT-bound there
INT_CEILING_GBS = 4110.0
METRIC = "routed requests/sec (prefix-match+evict+route) at 1/2/4/8 B200; % HBM peak"
UNIT = "requests/s"

DEFAULTS = {  # per workload: requests per burst per GPU, replicas, models, kv, l2
    "bursty": dict(requests=125_000, replicas=256, models=8, kv=100_000, l2=200_000),
    "long_context": dict(requests=12_500, replicas=64, models=1, kv=141_000, l2=200_000),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="bursty", choices=list(DEFAULTS))
    ap.add_argument("--requests", type=int, default=0, help="requests per burst per GPU")
    ap.add_argument("--replicas", type=int, default=0)
    ap.add_argument("--models", type=int, default=0)
    ap.add_argument("--kv", type=int, default=0)
    ap.add_argument("--l2", type=int, default=0)
    ap.add_argument("--block", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--check", type=int, default=0,
                    help="parity: K full-size bursts on the GPU and through the reference")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sample", type=int, default=0,
                    help="reference arm / cpu_baseline: requests per burst (bounded prefix)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no baselines)")
    ap.add_argument("--split-min", type=int, default=-1,
                    help="K1: prompts of >= this many tokens are split tasks (0 = never, "
                         "-1 = from the batch's token count)")
    ap.add_argument("--k1-after", default="auto", choices=["auto", "start", "staged"],
                    help="K1 of burst k+1 starts with step k (start) or once step k's K2 is "
                         "done (staged: K2 runs alone, K1 overlaps the latency-bound K3 / "
                         "admission); auto: start at N = 1, staged at N > 1")
    ap.add_argument("--k1-grid", default="auto",
                    choices=["auto", "persistent", "tasks", "tasks1"],
                    help="K1 grid: persistent CTAs, or one task per warp (CTAs retire so the "
                         "step's kernels interleave; tasks1: at most one K1 CTA per SM); "
                         "auto: tasks1 (persistent for config 3)")
    ap.add_argument("--k1-memo", default="off", choices=["on", "off"],
                    help="K1 prefix memo of shared leading tokens (pyg_set_hash_memo)")
    ap.add_argument("--k1-gate", default="off", choices=["on", "off"],
                    help="K1 of the next burst pauses while the step's admission runs "
                         "(pyg_set_hash_gate)")
    ap.add_argument("--free-sms", type=int, default=None,
                    help="K1 of step k+1 overlaps step k on a second stream, its grid capped at "
                         "(SMs - free_sms); -1 = no overlap (serial step)")
    a = ap.parse_args()
    # measured best per GPU count: K1 of the next burst on retiring CTAs, one
    # per SM -- from the step's start on one GPU, after the step's K2 on several (the sharded
    # step's cross-rank phases suffer most beside K1)
    # config 3 (few, long prompts): a persistent K1 spread over all but 48 SMs, from the
    # step's start, leaves the step's kernels SMs of their own
    multi = a.gpus > 1 or int(os.environ.get("WORLD_SIZE", "1")) > 1
    lc = a.workload == "long_context" and not multi
    if a.k1_after == "auto":
        a.k1_after = "staged" if multi else "start"
    if a.k1_grid == "auto":
        a.k1_grid = "persistent" if lc else "tasks1"
    if a.free_sms is None:
        a.free_sms = 48 if lc else 8
    for k, v in DEFAULTS[a.workload].items():
        if not getattr(a, k):
            setattr(a, k, v)
    return a


def maybe_self_launch(args):
    """bench.py --gpus N without torchrun: relaunch as N ranks (one process per GPU)."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
               str(port), os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)


# the step's stream outranks K1's (0): CTAs of its kernels are dispatched first as SMs free
STEP_PRIORITY = int(os.environ.get("PYG_STEP_PRIORITY", "-1"))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [[x.strip() for x in line.split(",")] for line in out.strip().splitlines()]
        rows = [r for r in rows if len(r) == 6]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        busy = [x for x in sm if x > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ------------------------------------------------------------------ workload
def setup_cluster(args):
    from paper_2604_25899_b200 import workload as W
    return W.make_cluster(args.replicas, args.models, kv=args.kv, l2=args.l2, seed=0)


def warm_inputs(args, cl, device):
    """The warm trace, its ops and the warm-fill plan (identical for every arm)."""
    from paper_2604_25899_b200 import steady as S
    n = 64 * args.replicas if args.workload == "bursty" else 4 * args.replicas
    warm = S.make_burst(10_000, n, args.seed + 17, device, args.workload, args.models)
    l2g = 64 if args.workload == "bursty" else 8
    ops = S.warm_ops(warm, cl, l3_prefixes=128 if args.workload == "bursty" else 16,
                     l2_per_group=l2g, seed=args.seed)
    off, placed = S.warm_fill_plan(warm, cl)
    return warm, ops, off, placed


def describe(args, ws):
    if args.workload == "bursty":
        return (f"config-4 bursty multi-LLM trace in bursts of {args.requests} requests per GPU "
                f"({ws * args.requests} per step; 8 steps x 125k = the config's 1M requests at N=1), "
                f"L~lognormal(2048, cv 1) in [64, 32768], 512 shared prefixes, 10% unprofiled, "
                f"{args.replicas} replicas ({args.models} models x {args.replicas // args.models}), "
                f"B={args.block}, kv={args.kv}, l2={args.l2}; state carried across bursts "
                f"(placements held 2 bursts, releases, warm-filled L1 -> eviction, ordered L3)")
    return (f"config-3 long-context mix in bursts of {args.requests} requests per GPU: "
            f"L=32768 (2048 role sys + 28672 carried context + 2048 unique), {args.replicas} "
            f"replicas, kv={args.kv} (capacity_holds binds), B={args.block}, l2={args.l2}; state "
            f"carried across bursts")


def algorithmic_bytes(bursts_host, B, cl, stats, max_cand):
    """SURVEY.md 8(d) bytes of the timed steps: K1 (8L + 8 ceil(L/B) + 16 per request), K2
    (32 B per probe of the per-candidate walks the reference semantics require: staged/B + 1
    per (request, candidate)), K3 (32 + 24 per request), admission (64 B per inserted block +
    32 B per lookup probe on 3 tiers), eviction (24 B per scanned L1 block + 8 per victim)."""
    tot = {"hash": 0, "staged": 0, "route": 0, "admit": 0, "evict": 0, "probes": 0}
    for tok_off, group, staged, placed in bursts_host:
        L = np.diff(tok_off)
        nb = (L + B - 1) // B
        tot["hash"] += 8 * int(L.sum()) + 8 * int(nb.sum()) + 16 * (len(L) + 1)
        ncand = np.diff(cl.cand_off)[group]
        mask = np.arange(max_cand)[None, :] < ncand[:, None]
        probes = int(((staged + B - 1) // B + 1)[mask].sum())
        tot["probes"] += probes
        tot["staged"] += 32 * probes + 4 * int(mask.sum())
        tot["route"] += 56 * len(L)
        tot["admit"] += int(sum(32 * 3 * (nb[r] // 4 + 1) + 64 * nb[r] for r in placed))
    blocks_per_l1 = float(np.mean(cl.kv_capacity)) / B
    tot["evict"] = int(24 * stats["evictions"] * blocks_per_l1 + 8 * stats["evicted_blocks"])
    tot["total"] = sum(tot[k] for k in ("hash", "staged", "route", "admit", "evict"))
    return tot


# --------------------------------------------------------------- reference arm
def reference_run(args, n_steps, n_warm, threads, hash_once, sample, seconds=None):
    """The reference through the burst sequence: warm state as ours, then bursts 0.. each
    truncated to its first `sample` requests.  Returns (requests, seconds) of the measured
    steps (those after n_warm), stopping early once `seconds` elapse."""
    from oracle.steady_ref import RefSteady
    from paper_2604_25899_b200 import steady as S
    cl = setup_cluster(args)
    warm, ops, off, placed = warm_inputs(args, cl, "cpu")
    ref = RefSteady(args.block, cl, threads=threads, hash_once=hash_once)
    ref.warm(warm, ops, off, placed)
    done, el = 0, 0.0
    for k in range(n_warm + n_steps):
        tr = S.make_burst(k, args.requests, args.seed, "cpu", args.workload, args.models,
                          n_keep=sample)
        toks = tr.tokens_np()
        rw, rm = S.registry_pairs(tr.wf, tr.role)
        t0 = time.perf_counter()
        ref.step(k, toks, tr.tok_off, tr.res, tr.group, tr.wf, tr.role, rw, rm, 1.0 + k,
                 S.hold_of(k, args.requests, tr.R))
        dt = time.perf_counter() - t0
        if k >= n_warm:
            done += tr.R
            el += dt
            if seconds is not None and el >= seconds:
                break
    return done, el, float(np.diff(tr.tok_off).mean())


def cpu_sample_desc(args, n, threads, hash_once, mean_len, sample):
    how = ("chain_boundary_hashes once + tier(L2).matched_prefix per candidate (hash-once)"
           if hash_once else "cache.lookup(prompt, nullptr).l2 per candidate (the engine's "
           "node_view, one rehash per candidate)")
    return (f"{n} requests = the first {sample} of each {args.workload} burst (same seeds, "
            f"cluster, warm state; state carried across the sample bursts), mean prompt "
            f"{mean_len:.0f} tokens, through the unmodified reference "
            f"(oracle/_ref/libpythia_ref{args.block}.so pref_burst: {how}, route, admission "
            f"with evict_for_space, releases) on {args.replicas} replicas, {threads} thread(s); "
            f"CPU {cpu_model()}")


def cpu_baseline(args, hash_once=False):
    from oracle.py_oracle import reference_available
    if not reference_available(args.block):
        return None
    sample = args.sample or (1000 if args.workload == "bursty" else 100)
    n, el, ml = reference_run(args, 50, 1, 1, hash_once, sample, args.cpu_seconds)
    return {"value": n / el, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": cpu_sample_desc(args, n, 1, hash_once, ml, sample)}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle.py_oracle import reference_available
    if not reference_available(args.block):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    cores = os.cpu_count() or 1
    sample = args.sample or (4000 if args.workload == "bursty" else 200)
    n, el, ml = reference_run(args, args.steps, args.warmup, cores, False, sample)
    value = n / el
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * el / max(args.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": describe(args, 1) + " [bounded prefix sample per burst]",
                       "replicas": args.replicas, "block_tokens": args.block,
                       "route_mode": "seq_commit", "sample_requests_per_burst": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": cpu_sample_desc(args, n, cores, False, ml, sample)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
class Arm:
    """One GPU's state for the steady-state bench: bursts in HBM, the cluster ctx, the
    hashing ctx on its own stream."""

    def __init__(self, args, dev, n_bursts):
        import ctypes
        import torch
        from paper_2604_25899_b200 import Context
        from paper_2604_25899_b200 import steady as S
        self.args, self.dev, self.S = args, dev, S
        self.cl = setup_cluster(args)
        cl = self.cl
        self.ctx = Context(cl.n_replicas, cl.kv_capacity, cl.l2_capacity, args.block,
                           device=dev.index)
        torch.cuda.set_stream(torch.cuda.Stream(device=dev, priority=STEP_PRIORITY))
        self.S_stream = torch.cuda.current_stream(dev)
        from paper_2604_25899_b200 import batch as PB
        self.PB = PB
        PB.bind_current_stream(self.ctx)
        warm, ops, off, placed = warm_inputs(args, cl, dev)
        self.n_fill = S.apply_warm_fill_gpu(self.ctx, warm, off, placed, args.block, dev)
        S.apply_ops_gpu(self.ctx, warm, ops)
        del warm
        self.bursts = []
        for k in range(n_bursts):
            tr = S.make_burst(k, args.requests, args.seed, dev, args.workload, args.models)
            self.bursts.append(S.upload_burst(tr, args.block, dev, k))
            del tr
        self.st = S.Steady(self.ctx, cl, args.requests, dev)
        self.st.reserve(self.bursts)
        self.overlap = args.free_sms >= 0
        self.H = torch.cuda.Stream(device=dev, priority=0) if self.overlap else self.S_stream
        self.hctx = Context(0, [], [], args.block, device=dev.index)
        self.hctx.set_stream(ctypes.c_void_p(self.H.cuda_stream))
        if self.overlap:
            n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
            self.hctx.set_hash_ctas(max(1, n_sm - args.free_sms))
        self.hctx.set_hash_split(args.split_min)
        self.hctx.set_hash_grid(args.k1_grid)
        self.hctx.set_hash_memo(args.k1_memo == "on")
        if self.overlap and args.k1_gate == "on":
            self.hctx.set_hash_gate(self.ctx)
        self.ev_h = {}
        torch.cuda.synchronize(dev)
        self.ctx.check_device_error()

    def launches(self):
        return self.ctx.kernel_launches() + self.hctx.kernel_launches()

    def hash_into(self, k, hev=None):
        import torch
        self.H.wait_stream(self.S_stream)  # K1(k) starts with step k-1 (step k-2 is done)
        if hev is not None:
            hev[0].record(self.H)
        self.PB.hash_batch(self.hctx, self.bursts[k].b)
        if hev is not None:
            hev[1].record(self.H)
        e = torch.cuda.Event()
        e.record(self.H)
        self.ev_h[k] = e

    def run(self, k0, n, evs=None, hevs=None, carry=False):
        """steps k0 .. k0+n-1.  K1 of burst k+1 overlaps step k; K1 of burst k0 runs first
        unless an earlier carry=True call launched it (the pipeline is already full), and
        with carry=True the last step launches K1 of burst k0+n.  hevs[i]: K1 of burst
        k0+i+1 (carry) / of burst k0+i."""
        fill = k0 not in self.ev_h
        if fill:
            self.hash_into(k0, hevs[0] if (hevs and not carry) else None)
        after_staged = self.args.k1_after == "staged"
        for i in range(n):
            k = k0 + i
            self.S_stream.wait_event(self.ev_h.pop(k))
            nxt = None
            if i + 1 < n or carry:
                j = i if carry else i + 1
                nxt = (lambda kk=k + 1, jj=j: self.hash_into(kk, hevs[jj] if hevs else None))
                if not after_staged:
                    nxt()
                    nxt = None
            e = evs[i] if evs else None
            if e:
                e[0].record(self.S_stream)
            self.PB.bind_current_stream(self.ctx)
            self.st.complete(self.bursts, k)
            self.st.compose_nodes(self.bursts[k - 1] if k >= 1 else None, k)
            self.st.registry(self.bursts[k])
            self.st.route_admit(self.bursts[k], k, 1.0 + k, e[1:] if e else None, nxt)


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        return run_sharded(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.check:
        return run_check(args, dev)
    W_, K = args.warmup, args.steps
    E = 0 if (args.no_e2e or args.profile) else args.e2e_steps
    arm = Arm(args, dev, W_ + K + 1)
    ctx = arm.ctx
    # warm-up fills the pipeline: its last step already runs K1 of the first timed burst, and
    # every timed step runs K1 of the burst after it (the last one's inside the timed span)
    arm.run(0, W_, carry=True)
    torch.cuda.synchronize(dev)
    ctx.check_device_error()
    ctx.counters(reset=True)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    l0 = arm.launches()
    ET = torch.cuda.Event
    evs = [[ET(enable_timing=True) for _ in range(5)] for _ in range(K)]
    hevs = [(ET(enable_timing=True), ET(enable_timing=True)) for _ in range(K)]
    t0, t1 = ET(enable_timing=True), ET(enable_timing=True)
    torch.cuda.synchronize(dev)
    t0.record(arm.S_stream)
    arm.run(W_, K, evs, hevs, carry=True)
    arm.S_stream.wait_stream(arm.H)  # the timed span ends after the last K1 too
    t1.record(arm.S_stream)
    torch.cuda.synchronize(dev)
    launches = arm.launches() - l0
    clk = clocks.stop()
    ctx.check_device_error()
    stats = ctx.counters(reset=True)
    ms = t0.elapsed_time(t1)
    ms_step = ms / K
    R = args.requests
    value = R * K / (ms / 1000.0)
    phases = ["bookkeeping", "staged", "route", "admit"]
    phase_ms = {p: sum(e[i].elapsed_time(e[i + 1]) for e in evs) / K for i, p in enumerate(phases)}
    phase_ms["hash"] = sum(a.elapsed_time(b) for a, b in hevs) / K
    # bytes: K1 exactly per timed burst (host offsets); the staged / admission terms from the
    # last burst's outputs (still in the ring), eviction from the measured counters
    timed = arm.bursts[W_ + 1:W_ + K + 1]  # the bursts K1 hashed inside the timed span
    hash_bytes = float(np.mean([8 * int(b.tok_off[-1]) + 8 * b.b.n_hashes + 16 * (b.R + 1)
                                for b in timed]))
    o = arm.st.out(W_ + K - 1)
    h = o.host()
    last = arm.bursts[W_ + K - 1]
    placed_last = h["placed"][:h["placed_off"][-1]]
    ab = algorithmic_bytes([(last.tok_off, last.group, h["staged"][:R], placed_last)],
                           args.block, arm.cl, {"evictions": 0, "evicted_blocks": 0},
                           arm.st.nodes.max_cand)
    peak, peak_src = peaks()
    hash_gbs = hash_bytes / (phase_ms["hash"] / 1000.0) / 1e9
    ev = algorithmic_bytes([], args.block, arm.cl, stats, arm.st.nodes.max_cand)["evict"] / K
    step_bytes = hash_bytes + ab["staged"] + ab["route"] + ab["admit"] + ev
    step_gbs = step_bytes / (ms_step / 1000.0) / 1e9

    alone = k1_alone(arm, W_ + 1, hash_bytes, peak_of())
    e2e = None
    if E:
        e2e = run_e2e(args, arm, E, W_ + K)
    traffic = hash_traffic(args)
    cpu = cpu_h1 = None
    if not args.no_cpu_baseline and not args.profile:
        cpu = cpu_baseline(args, hash_once=False)
        cpu_h1 = cpu_baseline(args, hash_once=True)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": W_,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {
            "workload": describe(args, 1), "route_mode": "seq_commit",
            "requests_per_step": R, "tokens_per_step": int(sum(b.b.n_tokens for b in
                                                               arm.bursts[W_:]) / K),
            "distinct_bursts": True,
            "placed_per_step": stats["admissions"] / K,
            "admitted_per_step": stats["admitted"] / K,
            "evicted_blocks_per_step": stats["evicted_blocks"] / K,
            "evicted_tokens_per_step": stats["evicted_tokens"] / K,
            "evictions_per_step": stats["evictions"] / K,
            "l3_promoted_tokens_per_step": stats["l3_promoted_tokens"] / K,
            "warm_fill_admissions": arm.n_fill,
            "l2_flush": "none needed: every step reads a distinct burst (%.2f GB of tokens) "
                        "larger than the 126 MB L2" % (arm.bursts[-1].b.n_tokens * 8 / 1e9),
            "parallelism": "one GPU holds every replica",
            "k1_overlap": (f"K1 of burst k+1 on a second stream from step k's "
                           f"{'K2 end' if args.k1_after == 'staged' else 'start'}, "
                           f"{k1_grid_desc(args)}"
                           f"{', paused while the admission runs' if args.k1_gate == 'on' else ''}; "
                           "the timed span holds K steps and K K1 launches (bursts k0+1 .. "
                           "k0+K; burst k0's K1 ran in the last warm-up step, as in the steady "
                           "pipeline)")
            if arm.overlap else "none (serial)"},
        "roofline": {"bound": "hbm", "kernel": "k_hash_staged (K1, chain_boundary_hashes)",
                     "achieved": hash_gbs, "peak": peak, "unit": "GB/s", "frac": hash_gbs / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": int(hash_bytes),
                     "avg_launch_ms": phase_ms["hash"],
                     "note": ("avg_launch_ms is K1 inside the timed steps, sharing the GPU with "
                              "the step it overlaps; 'alone' is the same launch on an idle GPU"),
                     "alone": alone,
                     "int_ceiling": {"gbs": INT_CEILING_GBS, "frac": hash_gbs / INT_CEILING_GBS,
                                     "source": "profiles/r01_fnv_core.txt: FNV-1a core with "
                                               "register-resident tokens, 513 Gtok/s"}},
        "step_roofline": {"achieved": step_gbs, "frac": step_gbs / peak,
                          "algorithmic_bytes_per_step": int(step_bytes), "probes": ab["probes"]},
        "phase_ms": phase_ms, "clocks": clk, "gpu_launches": int(launches),
        "e2e": e2e, "cpu_baseline": cpu, "cpu_baseline_hash_once": cpu_h1,
    }
    print(json.dumps(line), flush=True)


def peak_of():
    return peaks()[0]


def k1_alone(arm, k, hash_bytes, peak, reps=5):
    """K1 (hash prep + k_hash_staged) of burst k re-run on an idle GPU after the timed span:
    median of `reps` launches, CUDA events on its stream."""
    import torch
    torch.cuda.synchronize(arm.dev)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(arm.H)
        arm.PB.hash_batch(arm.hctx, arm.bursts[k].b)
        b.record(arm.H)
        torch.cuda.synchronize(arm.dev)
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    gbs = hash_bytes / (ms / 1000.0) / 1e9
    return {"avg_launch_ms": ms, "achieved": gbs, "frac": gbs / peak}


def k1_grid_desc(args):
    return {"persistent": f"persistent grid of SMs - {args.free_sms} CTAs",
            "tasks": "one task per warp (CTAs retire as they finish)",
            "tasks1": "one task per warp, at most one K1 CTA per SM (CTAs retire as they "
                      "finish; the step's kernels take the SMs they free, higher stream "
                      "priority)"}[args.k1_grid]


def hash_traffic(args):
    """K1's DRAM bytes per launch from the committed ncu capture of this workload (ncu
    replays kernels, so it is not taken inside bench.py), else None."""
    prof = os.path.join(ROOT, "profiles", "hash_kernel_traffic.json")
    try:
        with open(prof) as f:
            d = json.load(f)
        if d.get("workload") == args.workload and args.requests == 125000:
            return d.get("traffic_bytes_per_launch")
    except Exception:
        pass
    return None


def run_e2e(args, arm, E, k_first):
    """E more steps through the public API from pinned host buffers: per step the burst's
    tokens, offsets and request metadata go host->device (copy stream, one burst ahead), K1
    and the step run, decisions / admissions / lookups come back (d2h stream)."""
    import torch
    S, PB = arm.S, arm.PB
    dev = arm.dev
    host, devb = [], []
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    for i in range(E):
        k = k_first + i
        tr = S.make_burst(k, args.requests, args.seed, dev, args.workload, args.models)
        b = S.upload_burst(tr, args.block, dev, k)  # device buffers (overwritten by the copies)
        rw, rm = S.registry_pairs(tr.wf, tr.role)
        host.append({"tokens": tr.tokens.cpu().pin_memory(), "tok_off": pin(tr.tok_off),
                     "res": pin(tr.res.view(np.int64).reshape(tr.R, 4)), "group": pin(tr.group),
                     "wf": pin(tr.wf), "role": pin(tr.role), "reg_wf": pin(rw),
                     "reg_mask": pin(rm.view(np.int64))})
        devb.append(b)
        del tr
    R = args.requests
    res_h = [[torch.empty((R, 3), dtype=torch.int64).pin_memory(),
              torch.empty(R, dtype=torch.int32).pin_memory(),
              torch.empty((R, 3), dtype=torch.int64).pin_memory()] for _ in range(2)]
    bursts = {k_first - 2 + j: arm.bursts[k_first - 2 + j] for j in range(2)}
    for i in range(E):
        bursts[k_first + i] = devb[i]
    cp = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    up = {}
    h2d_bytes = sum(int(v.numel() * v.element_size()) for v in host[0].values())
    d2h_bytes = sum(int(t.numel() * t.element_size()) for t in res_h[0])

    def upload(i):
        b, h = devb[i], host[i]
        with torch.cuda.stream(cp):
            b.b.tokens[:h["tokens"].numel()].copy_(h["tokens"], non_blocking=True)
            b.b.tok_off.copy_(h["tok_off"], non_blocking=True)
            b.b.res.copy_(h["res"], non_blocking=True)
            b.b.group.copy_(h["group"], non_blocking=True)
            b.b.wf.copy_(h["wf"], non_blocking=True)
            b.b.role.copy_(h["role"], non_blocking=True)
            b.reg_wf.copy_(h["reg_wf"], non_blocking=True)
            b.reg_mask.copy_(h["reg_mask"], non_blocking=True)
            e = torch.cuda.Event()
            e.record(cp)
            up[i] = e

    import ctypes
    from paper_2604_25899_b200 import _lib
    fetched = [None, None]
    def k1(i):
        """hash offsets + K1 of e2e burst i on the hash stream, after its upload"""
        b = devb[i]
        arm.H.wait_event(up.pop(i))
        _lib.check(_lib._lib.pyg_hash_offsets_dev(arm.hctx.h,
                                                  ctypes.c_void_p(b.b.tok_off.data_ptr()), b.R,
                                                  ctypes.c_void_p(b.b.hash_off.data_ptr()), None))
        PB.hash_batch(arm.hctx, b.b)
        e = torch.cuda.Event()
        e.record(arm.H)
        return e

    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    upload(0)
    if E > 1:
        upload(1)
    eh = k1(0)
    for i in range(E):
        k = k_first + i
        b = devb[i]
        arm.S_stream.wait_event(eh)
        PB.bind_current_stream(arm.ctx)
        arm.st.complete(bursts, k)
        arm.st.compose_nodes(bursts[k - 1], k)
        arm.st.registry(b)
        o = arm.st.route_admit(b, k, 1.0 + k)
        es = torch.cuda.Event()
        es.record(arm.S_stream)
        if i + 1 < E:          # K1 of the next burst overlaps this step
            eh = k1(i + 1)
        if i + 2 < E:
            upload(i + 2)
        s = i % 2
        with torch.cuda.stream(d2h):
            d2h.wait_event(es)
            if fetched[s] is not None:
                fetched[s].synchronize()
            res_h[s][0].copy_(o.decisions[:R], non_blocking=True)
            res_h[s][1].copy_(o.admitted[:R], non_blocking=True)
            res_h[s][2].copy_(o.match3[:R], non_blocking=True)
            ef = torch.cuda.Event()
            ef.record(d2h)
            fetched[s] = ef
    torch.cuda.synchronize(dev)
    el = time.perf_counter() - t0
    arm.ctx.check_device_error()
    return {"value": R * E / el, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes,
            "d2h_bytes_per_step": d2h_bytes, "ms_per_step": 1000.0 * el / E, "steps": E,
            "via": ("public API from pinned host buffers: per step the burst's tokens, offsets "
                    "and request metadata are copied host->device (copy stream, one burst "
                    "ahead), hash offsets + K1 + the steady step run on device, decisions / "
                    "admissions / lookups are copied back; wall clock over the steps")}


def run_check(args, dev):
    """--check K: K full-size bursts on the GPU and through the unmodified reference (all host
    threads for the staged values, hash-once -- the same reference functions without repeated
    hashing), compared burst by burst and, at the end, tier by tier."""
    import torch
    from oracle.steady_ref import RefSteady
    K = args.check
    t_start = time.perf_counter()
    arm = Arm(args, dev, K)
    S = arm.S
    cl = arm.cl
    ref = RefSteady(args.block, cl, threads=os.cpu_count() or 1, hash_once=True)
    warm, ops, off, placed = warm_inputs(args, cl, "cpu")
    ref.warm(warm, ops, off, placed)
    del warm
    report = {"check": "steady-state bursts vs the unmodified reference", "bursts": K,
              "workload": describe(args, 1), "per_burst": []}
    ok = True
    arm.ctx.counters(reset=True)
    for k in range(K):
        arm.run(k, 1)
        torch.cuda.synchronize(dev)
        arm.ctx.check_device_error()
        got = arm.st.out(k).host()
        b = arm.bursts[k]   # the reference gets the very same inputs
        toks = b.b.tokens.cpu().numpy().view(np.uint64)
        rw, rm = S.registry_pairs(b.wf, b.role)
        t0 = time.perf_counter()
        d, a, m3, stg = ref.step(k, toks, b.tok_off, b.res, b.group, b.wf, b.role, rw, rm,
                                 1.0 + k, b.hold_h, want_staged=True)
        t_ref = time.perf_counter() - t0
        R = b.R
        mc = stg.shape[1]
        gd = got["decisions"][:R]
        pl = d["target"] >= 0
        row = {"burst": k, "requests": R, "placed": int(pl.sum()), "admitted": int(a.sum()),
               "ref_seconds": round(t_ref, 2),
               "staged": bool(np.array_equal(got["staged"][:R, :mc], stg)),
               "target": bool(np.array_equal(gd["target"], d["target"])),
               "tiebreak": bool(np.array_equal(gd["tiebreak"], d["tiebreak"])),
               "headroom": bool(np.array_equal(gd["headroom"], d["headroom"])),
               "oom_bound_bits": gd["oom_bound"].tobytes() == d["oom_bound"].tobytes(),
               "admitted_eq": bool(np.array_equal(got["admitted"][:R], a)),
               "match3": bool(np.array_equal(got["match3"][:R][pl], m3[pl]))}
        row["ok"] = all(v for kk, v in row.items() if isinstance(v, bool))
        ok &= row["ok"]
        report["per_burst"].append(row)
        print(json.dumps(row), flush=True)
        del toks
    stats = arm.ctx.counters()
    tiers_ok = True
    bad = []
    for n in range(cl.n_replicas):
        for t in (0, 1):
            if arm.ctx.dump(n, t).tobytes() != ref.dump(n, t).tobytes():
                tiers_ok = False
                bad.append((n, t))
    l3_ok = arm.ctx.dump(0, 2).tobytes() == ref.dump(0, 2).tobytes()
    report.update({"tiers_equal": tiers_ok, "l3_equal": l3_ok, "bad_tiers": bad[:10],
                   "device_stats": stats, "ok": bool(ok and tiers_ok and l3_ok),
                   "seconds": round(time.perf_counter() - t_start, 1),
                   "host_threads": os.cpu_count()})
    print(json.dumps(report))


def run_e2e_sharded(args, sh, bursts, k_first, E, ws, rank, dev, Sst, H, hctx):
    """E more sharded steps through the public API from pinned host buffers, on every rank:
    its burst's tokens, offsets, request metadata and the burst's registry pairs go
    host->device (copy stream, one burst ahead), hash offsets + K1 and the sharded step run,
    its requests' decisions / admissions / lookups come back.  Wall clock per rank between
    barriers, max over ranks; value = all ranks' requests / that time."""
    import ctypes
    import torch
    import torch.distributed as dist
    from paper_2604_25899_b200 import _lib
    from paper_2604_25899_b200 import batch as PB
    R = args.requests
    r0, r1 = int(sh.plan.req_off[rank]), int(sh.plan.req_off[rank + 1])
    host, dst = [], []
    for i in range(E):
        b = bursts[k_first + i]
        rw, rm, _, _ = sh.reg[k_first + i]
        dv = {"tokens": b.b.tokens[:b.b.n_tokens], "tok_off": b.b.tok_off, "res": b.b.res,
              "group": b.b.group, "wf": b.b.wf, "role": b.b.role, "reg_wf": rw, "reg_mask": rm}
        dst.append(dv)
        host.append({k: v.cpu().pin_memory() for k, v in dv.items()})
    res_h = [[torch.empty((r1 - r0, 3), dtype=torch.int64).pin_memory(),
              torch.empty(R, dtype=torch.int32).pin_memory(),
              torch.empty((R, 3), dtype=torch.int64).pin_memory()] for _ in range(2)]
    h2d_bytes = sum(int(v.numel() * v.element_size()) for v in host[0].values())
    d2h_bytes = sum(int(t.numel() * t.element_size()) for t in res_h[0])
    cp = torch.cuda.Stream(device=dev)
    d2h = torch.cuda.Stream(device=dev)
    up = {}

    def upload(i):
        with torch.cuda.stream(cp):
            for key, v in host[i].items():
                dst[i][key].copy_(v, non_blocking=True)
            e = torch.cuda.Event()
            e.record(cp)
            up[i] = e

    def k1(i):
        b = bursts[k_first + i]
        H.wait_event(up.pop(i))
        _lib.check(_lib._lib.pyg_hash_offsets_dev(hctx.h, ctypes.c_void_p(b.b.tok_off.data_ptr()),
                                                  b.R, ctypes.c_void_p(b.b.hash_off.data_ptr()),
                                                  None))
        PB.hash_batch(hctx, b.b)
        e = torch.cuda.Event()
        e.record(H)
        return e

    fetched = [None, None]
    torch.cuda.synchronize(dev)
    dist.barrier()
    t0 = time.perf_counter()
    upload(0)
    if E > 1:
        upload(1)
    eh = k1(0)
    for i in range(E):
        k = k_first + i
        Sst.wait_event(eh)
        stp = sh.step(k, 1.0 + k)
        es = torch.cuda.Event()
        es.record(Sst)
        if i + 1 < E:          # K1 of the next burst overlaps this step
            eh = k1(i + 1)
        if i + 2 < E:
            upload(i + 2)
        s_ = i % 2
        with torch.cuda.stream(d2h):
            d2h.wait_event(es)
            if fetched[s_] is not None:
                fetched[s_].synchronize()
            res_h[s_][0].copy_(stp.decisions[r0:r1], non_blocking=True)
            res_h[s_][1].copy_(stp.out_adm[:R], non_blocking=True)
            res_h[s_][2].copy_(stp.out_m3[:R], non_blocking=True)
            ef = torch.cuda.Event()
            ef.record(d2h)
            fetched[s_] = ef
    torch.cuda.synchronize(dev)
    el = time.perf_counter() - t0
    sh.ctx.check_device_error()
    t = torch.tensor([el], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    el = float(t[0].item())
    return {"value": R * ws * E / el, "unit": UNIT, "h2d_bytes_per_step": h2d_bytes * ws,
            "d2h_bytes_per_step": d2h_bytes * ws, "ms_per_step": 1000.0 * el / E, "steps": E,
            "via": ("public API from pinned host buffers on every rank: per step each GPU's "
                    "burst (tokens, offsets, request metadata, registry pairs) is copied "
                    "host->device (copy stream, one burst ahead), hash offsets + K1 + the "
                    "sharded step run, its requests' decisions / admissions / lookups are "
                    "copied back; wall clock between barriers, max over ranks; byte counts "
                    "summed over the GPUs")}


def run_sharded(args):
    """N > 1 (one process per GPU): the cluster's replicas split by model over the GPUs
    (steady_shard.py), every rank brings its own burst of args.requests per step (weak
    scaling); value = all ranks' routed requests / the max over ranks of the timed span."""
    import ctypes
    import torch
    import torch.distributed as dist
    from paper_2604_25899_b200 import Context
    from paper_2604_25899_b200 import batch as PB
    from paper_2604_25899_b200 import steady as S
    from paper_2604_25899_b200.steady_shard import ShardedSteady
    ws, rank, local = dist_env()
    dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    W_, K = args.warmup, args.steps
    cl = setup_cluster(args)
    per = cl.n_replicas // ws
    lo, hi = rank * per, (rank + 1) * per
    ctx = Context(per, cl.kv_capacity[lo:hi], cl.l2_capacity[lo:hi], args.block, device=local)
    Sst = torch.cuda.Stream(device=dev, priority=STEP_PRIORITY)
    torch.cuda.set_stream(Sst)
    PB.bind_current_stream(ctx)
    warm, ops, off, placed = warm_inputs(args, cl, dev)
    loc_off = (off[lo:hi + 1] - off[lo]).astype(np.int32)
    n_fill = S.apply_warm_fill_gpu(ctx, warm, loc_off, placed[off[lo]:off[hi]], args.block, dev)
    S.apply_ops_gpu(ctx, warm, ops, rep_base=lo)
    del warm
    E = 0 if (args.no_e2e or args.profile) else args.e2e_steps
    bursts = []
    for k in range(W_ + K + 1 + E):
        tr = S.make_burst(k * ws + rank, args.requests, args.seed, dev, args.workload,
                          args.models)
        bursts.append(S.upload_burst(tr, args.block, dev, k * ws + rank))
        del tr
    sh = ShardedSteady(ctx, cl, rank, ws, bursts, args.block, dev)
    sh.reserve()
    sh.build_directory()
    H = torch.cuda.Stream(device=dev, priority=0)
    hctx = Context(0, [], [], args.block, device=local)
    hctx.set_stream(ctypes.c_void_p(H.cuda_stream))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    hctx.set_hash_ctas(max(1, n_sm - args.free_sms))
    hctx.set_hash_split(args.split_min)
    hctx.set_hash_grid(args.k1_grid)
    hctx.set_hash_memo(args.k1_memo == "on")
    if args.k1_gate == "on":
        hctx.set_hash_gate(ctx)
    ev_h = {}

    def hash_into(k, hev=None):
        H.wait_stream(Sst)
        if hev is not None:
            hev[0].record(H)
        PB.hash_batch(hctx, bursts[k].b)
        if hev is not None:
            hev[1].record(H)
        e = torch.cuda.Event()
        e.record(H)
        ev_h[k] = e

    def run(k0, n, hevs=None, pevs=None, carry=False):
        # as Arm.run: K1 of burst k+1 overlaps step k; with carry the pipeline stays full
        if k0 not in ev_h:
            hash_into(k0, hevs[0] if (hevs and not carry) else None)
        for i in range(n):
            k = k0 + i
            Sst.wait_event(ev_h.pop(k))
            nxt = None
            if i + 1 < n or carry:
                j = i if carry else i + 1
                nxt = (lambda kk=k + 1, jj=j: hash_into(kk, hevs[jj] if hevs else None))
                if args.k1_after != "staged":
                    nxt()
                    nxt = None
            sh.step(k, 1.0 + k, ev=pevs[i] if pevs is not None else None, after_staged=nxt)

    run(0, W_, carry=True)
    torch.cuda.synchronize(dev)
    ctx.check_device_error()
    ctx.counters(reset=True)
    dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    l0 = ctx.kernel_launches() + hctx.kernel_launches()
    ET = torch.cuda.Event
    hevs = [(ET(enable_timing=True), ET(enable_timing=True)) for _ in range(K)]
    t0, t1 = ET(enable_timing=True), ET(enable_timing=True)
    pevs = [dict() for _ in range(K)]
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0.record(Sst)
    run(W_, K, hevs, pevs, carry=True)
    Sst.wait_stream(H)  # the timed span ends after the last K1 too
    t1.record(Sst)
    torch.cuda.synchronize(dev)
    names = ["begin", "start", "staged", "exchange", "route", "pull+admit", "l3_chain", "lists"]
    phase_ms = {("bookkeeping" if a == "begin" else b): sum(p[a].elapsed_time(p[b]) for p in pevs) / K
                for a, b in zip(names[:-1], names[1:])}
    phase_ms.pop("start", None)
    launches = ctx.kernel_launches() + hctx.kernel_launches() - l0
    clk = clocks.stop()
    ctx.check_device_error()
    st = ctx.counters(reset=True)
    ms = t0.elapsed_time(t1)
    e2e = run_e2e_sharded(args, sh, bursts, W_ + K, E, ws, rank, dev, Sst, H, hctx) if E else None
    hash_ms = sum(a.elapsed_time(b) for a, b in hevs) / K
    t = torch.tensor([ms, hash_ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, hash_ms_max = float(t[0].item()), float(t[1].item())
    cnt = torch.tensor([st["admissions"], st["admitted"], st["evicted_blocks"], launches],
                       dtype=torch.int64, device=dev)
    dist.all_reduce(cnt)
    timed = bursts[W_ + 1:W_ + K + 1]  # the bursts K1 hashed inside the timed span
    hash_bytes = float(np.mean([8 * int(b.tok_off[-1]) + 8 * b.b.n_hashes + 16 * (b.R + 1)
                                for b in timed]))
    hash_gbs = hash_bytes / (hash_ms / 1000.0) / 1e9
    peak, peak_src = peaks()
    R_tot = args.requests * ws
    value = R_tot * K / (ms_max / 1000.0)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K,
            "warmup": W_, "ms_per_step": ms_max / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {
                "workload": describe(args, ws), "route_mode": "seq_commit",
                "requests_per_step": R_tot, "requests_per_step_per_gpu": args.requests,
                "distinct_bursts": True,
                "placed_per_step": int(cnt[0].item()) / K,
                "admitted_per_step": int(cnt[1].item()) / K,
                "evicted_blocks_per_step": int(cnt[2].item()) / K,
                "warm_fill_admissions_rank0": n_fill,
                "l2_flush": "none needed: every step reads distinct bursts larger than the L2",
                "parallelism": (f"{ws} GPUs, replicas split by model ({per} per GPU, models "
                                f"{sh.own} on rank 0): K1/K2 on the origin GPU, route rows "
                                "over NVLink peer memory (flag barrier), K3 per model on its "
                                "owner, placed requests pulled by the owner over NVLink, L3 "
                                "promotions chained over the ranks in engine order"),
                "k1_overlap": (f"K1 of burst k+1 on a second stream from step k's "
                               f"{'K2 end' if args.k1_after == 'staged' else 'start'}, "
                               f"{k1_grid_desc(args)}; the timed span holds K steps and K K1 "
                               "launches (bursts k0+1 .. k0+K; burst k0's K1 ran in the last "
                               "warm-up step)")},
            "roofline": {"bound": "hbm", "kernel": "k_hash_staged (K1), rank 0",
                         "achieved": hash_gbs, "peak": peak, "unit": "GB/s",
                         "frac": hash_gbs / peak, "traffic": hash_traffic(args),
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": int(hash_bytes),
                         "avg_launch_ms": hash_ms, "max_over_ranks_launch_ms": hash_ms_max},
            "phase_ms_rank0": phase_ms, "hash_ms_rank0": hash_ms,
            "clocks": clk, "gpu_launches": int(cnt[3].item()), "e2e": e2e,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    # NCCL's banner would be a second stdout line next to the JSON line
    if os.environ.get("NCCL_DEBUG", "").upper() in ("VERSION", "INFO", "TRACE"):
        os.environ["NCCL_DEBUG"] = "WARN"
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    maybe_self_launch(args)
    run_ours(args)


if __name__ == "__main__":
    main()
