#!/usr/bin/env python
"""Training events/sec of the DistTGL training step on B200 (BASELINE.json metric).

One "step" = one barrier of the i x j x k schedule: every rank runs one
sub-iteration over its 600-event slice (sample -> plan -> memory read -> GRU
freshen -> attention -> decoder/BCE -> backward -> root writes -> gradient
all-reduce -> Adam). N=1 runs BASELINE configs[1] (Reddit shape, TGN + static
memory); N>1 runs the same workload with memory parallelism k=N, one GPU per
trainer, weak scaling (epochs=N so every memory copy sweeps a full epoch).
--config c3 / c4 run BASELINE configs[2] / [3] with mini-batch (i=N) / epoch
(j=N) parallelism instead; c5p / c5 the GDELT shape (5M prefix / full stream).
The timed window is mid-stream: the run is fast-forwarded so the K timed
barriers are centred on the middle of the schedule, where the CPU reference
legs are timed as well; the line reports both windows.
`--impl reference` (rank 0 only) times the unmodified reference trainer
(oracle/_ref) on all the host cores: for k-parallel configs (1,1,G) with G =
one memory group per two CPUs (>= N), plus its (1,1,N) number as
`same_parallelism`; for c3 / c4 the B200 arm's own (i,j,k).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training events/sec (device-timed, max over ranks)"
CONFIGS = {
    # BASELINE.json configs[1]: Reddit shape, TGN + static node memory
    "c2": dict(workload="synthetic Reddit-shape CTDG (C2): 10,984 nodes, 672,447 events, "
                        "172-d edge feats, TGN + static memory, 10 recent nbrs, mem 100, batch 600",
               nodes=10984, events=672447, d_e=172, d_static=100),
    "c1": dict(workload="synthetic Wikipedia-shape CTDG (C1): 9,227 nodes, 157,474 events, "
                        "172-d edge feats, TGN, 10 recent nbrs, mem 100, batch 600",
               nodes=9227, events=157474, d_e=172, d_static=0),
    "c5p": dict(workload="synthetic GDELT-shape CTDG (C5, 5M-event prefix): 16,682 nodes, "
                         "186-d edge feats, TGN + static memory, batch 600",
                nodes=16682, events=5_000_000, d_e=186, d_static=100),
    # BASELINE.json configs[2]: LastFM shape, high-degree, mini-batch parallelism i = N
    "c3": dict(workload="synthetic LastFM-shape CTDG (C3): 1,980 nodes, 1,293,103 events, no edge feats, "
                        "TGN + static memory, 10 recent nbrs, mem 100, local batch 600, mini-batch parallelism i=N",
               nodes=1980, events=1_293_103, d_e=0, d_static=100, axis="i"),
    # BASELINE.json configs[3]: MOOC shape, epoch parallelism j = N
    "c4": dict(workload="synthetic MOOC-shape CTDG (C4): 7,144 nodes, 411,749 events, no edge feats, "
                        "TGN + static memory, 10 recent nbrs, mem 100, local batch 600, epoch parallelism j=N",
               nodes=7144, events=411_749, d_e=0, d_static=100, axis="j"),
    # SURVEY 8(d) C5 variant: the paper's global batch of 3200 events per trainer
    "c5p3200": dict(workload="synthetic GDELT-shape CTDG (C5, 5M-event prefix), local batch 3200 "
                             "(the paper's batch, SURVEY 8(d)): 16,682 nodes, 186-d edge feats, TGN + static memory",
                    nodes=16682, events=5_000_000, d_e=186, d_static=100, batch=3200),
    # BASELINE.json configs[4] at full size: 191M events x 186 fp32 features
    # (143 GB) streamed into HBM by the chunked generator
    "c5": dict(workload="synthetic GDELT-shape CTDG (C5): 16,682 nodes, 191,290,882 events, "
                        "186-d edge feats, TGN + static memory, batch 600",
               nodes=16682, events=191_290_882, d_e=186, d_static=100),
}
LOCAL_BATCH = 600  # default local batch (BASELINE configs); a config may set "batch"


def batch_of(cfg):
    return cfg.get("batch", LOCAL_BATCH)
TRAIN_FRAC = 0.70
REF_MAX_EVENTS = 5_000_000  # f64 host copy of a GDELT-shape prefix: ~7.5 GB


def model_dims(cfg):
    return dict(d_mem=100, d_time=100, d_static=cfg["d_static"], d_attn=100, d_hidden=100,
                n_neighbors=10)


# ----------------------------------------------------------------- roofline bookkeeping
def attn_proj_flops(sz, cfg):
    """Algorithmic FLOPs of the attention projection GEMMs (node / edge split,
    SURVEY 8(a) a8 by linearity): per pair the edge part [e | cos(dt w) | 1] ->
    K|V, per support the node part [s_hat | static] -> Q|K|V:
    2 * (P * (d_e + d_t + 1) * 2 d_a + U * (d + d_s) * 3 d_a)."""
    d, ds, de, dt, da = 100, cfg["d_static"], cfg["d_e"], 100, 100
    return 2.0 * (sz["P"] * (de + dt + 1) * 2 * da + sz["U"] * (d + ds) * 3 * da)


def attn_proj_bytes(sz, cfg):
    """Compulsory bytes of those launches in fp32-equivalents (a bf16 hi/lo
    pair is 4 bytes): the edge rows EF [P x (d_e + d_t + 1)] and node rows NF
    [U x (d + d_s)] in, K|V edge parts [P x 2 d_a] and node parts [U x 3 d_a]
    out. (Weights are L2-resident and excluded.)"""
    d, ds, de, dt, da = 100, cfg["d_static"], cfg["d_e"], 100, 100
    return 4.0 * (sz["P"] * (de + dt + 1 + 2 * da) + sz["U"] * (d + ds + 3 * da))


def step_model_flops(sz, cfg):
    """SURVEY.md 8(d) model FLOPs of one sub-iteration (forward + dW + dX ~ 3x
    forward MACs x 2): KV, Q, GRU and decoder contractions."""
    d, ds, de, dt, da, dh = 100, cfg["d_static"], cfg["d_e"], 100, 100, 100
    q_in, kv_in, gin = d + ds + dt, d + ds + de + dt, 3 * d + dt + de
    macs = (2 * sz["P"] * kv_in * da + sz["R"] * q_in * da + sz["U"] * (3 * d * gin)
            + 2 * sz["B"] * 2 * da * dh)
    return 6.0 * macs


def ijk_of(cfg, world):
    """The B200 arm's (i, j, k): the config's parallelism axis carries the N ranks."""
    ax = cfg.get("axis", "k")
    return (world, 1, 1) if ax == "i" else (1, world, 1) if ax == "j" else (1, 1, world)


def step_compulsory_bytes(sz, cfg, nparam):
    """SURVEY.md 8(d) compulsory fp32 traffic of one sub-iteration: sampler
    probes R n (t f64 + event + neighbour), memory + mail rows of the U
    supports (1,220 B each), their static rows, edge-feature rows of the P
    pairs and U mails, the W root-write rows, and dense Adam (28 B/param) plus
    gradient zeroing (4 B/param)."""
    d_s, d_e = cfg["d_static"], cfg["d_e"]
    return (sz["R"] * 10 * 16 + sz["U"] * 1220 + sz["U"] * d_s * 4 + (sz["P"] + sz["U"]) * d_e * 4
            + sz["W"] * 1220 + 32 * nparam)


def step_roofline(sz, cfg, nparam, events_s_per_gpu, peaks):
    """Step-level roofline: t_roof per training event =
    max(model FLOPs / bf16 peak, compulsory bytes / HBM peak), from the
    mid-stream plan sizes measured in this run."""
    B = max(sz["B"], 1)
    f_ev = step_model_flops(sz, cfg) / B
    b_ev = step_compulsory_bytes(sz, cfg, nparam) / B
    t_t = f_ev / (peaks["bf16_tflops"] * 1e12)
    t_h = b_ev / (peaks["hbm_gbs"] * 1e9)
    t_roof = max(t_t, t_h)
    return {"bound": "tensor" if t_t >= t_h else "hbm", "mflop_per_event": f_ev / 1e6,
            "kb_per_event": b_ev / 1e3, "t_roof_ns_per_event": t_roof * 1e9,
            "roofline_events_s_per_gpu": 1.0 / t_roof, "achieved_events_s_per_gpu": events_s_per_gpu,
            "frac": events_s_per_gpu * t_roof}


def roofline_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of the roofline kernel (the
    tc_gemm_kernel group) from the committed ncu --set full capture of one
    barrier's GEMM launches (profiles/r02b_roofline_traffic.json, else the
    round-2 capture), per launch."""
    p = os.path.join(ROOT, "profiles", "r02b_roofline_traffic.json")
    if not os.path.exists(p):
        p = os.path.join(ROOT, "profiles", "r02_roofline_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d["dram_bytes_per_launch"]


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = list(self.rows)
        if not rows:  # region too short for the sampler: take one reading now
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits", "-i", str(self.device)],
                                     capture_output=True, text=True, timeout=10).stdout
                rows = [[p.strip() for p in out.strip().split(",")]]
            except Exception:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(self.rows)}


# ----------------------------------------------------------------- reference (CPU) arm
_REF_GRAPHS: dict = {}


def reference_time(cfg, ijk, barriers, warmup, log=print):
    """Times the unmodified reference (oracle/_ref, compiled from
    /root/reference/proj/include by oracle/Makefile) on this host's cores:
    run_sequential at (1,1,1), run_training (threaded: one thread per trainer
    plus one daemon per memory copy) otherwise, on the mid-stream window that
    starts at the middle of the training range (the B200 arm's timed window is
    centred there too). Returns (events/s, seconds, events, threads, window)."""
    from oracle import ref
    from oracle import tgnn_oracle as O

    i, j, k = ijk
    t0 = time.time()
    # the generator is sequential, so a prefix of the stream is the full
    # stream's prefix: the f64 reference holds at most REF_MAX_EVENTS of it
    n_ev = min(cfg["events"], REF_MAX_EVENTS)
    key = (cfg["nodes"], n_ev, cfg["d_e"])
    if key not in _REF_GRAPHS:  # one generated graph per workload and process
        g = ref.RefGraph.synthetic(cfg["nodes"], n_ev, d_e=cfg["d_e"], seed=1)
        _REF_GRAPHS[key] = (g, g.export(feats=False)[2])
        log(f"[ref] graph ready in {time.time() - t0:.1f}s")
    g, t = _REF_GRAPHS[key]
    mc = O.ModelConfig(d_e=cfg["d_e"], num_nodes=cfg["nodes"], max_t=float(t[-1]), **model_dims(cfg))
    mid = int(n_ev * TRAIN_FRAC) // 2
    out = None
    for phase, nbar in (("warmup", warmup), ("timed", barriers)):
        if nbar <= 0:
            continue
        lo = mid
        hi = lo + nbar * batch_of(cfg) * i * k
        tc = ref.train_cfg(i=i, j=j, k=k, local_batch=batch_of(cfg), seed=1, epochs=j, lr_base=1e-3)
        r = g.run(mc, tc, lo, hi, want_params=False)
        if phase == "timed":
            ev = int(ref.assignment(tc, lo, hi)["traversed_after"][-1])
            threads = i * j * k + (k if i * j * k > 1 else 0)
            out = (ev / r["elapsed_s"], r["elapsed_s"], ev, threads, [lo, hi])
        mid = hi
    return out


def reference_arm(args, world, rank, emit):
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    from oracle import ref
    if not ref.available():
        emit({"impl": "reference", "unavailable": "oracle/_ref not built"})
        return 0
    # bound the sample: each reference barrier is several seconds of CPU work
    steps = min(args.steps, args.ref_max_steps)
    warm = min(args.warmup, 1)
    log = lambda *a: print(*a, file=sys.stderr)  # noqa: E731
    ours = ijk_of(cfg, world)
    if cfg.get("axis", "k") == "k":
        # all the host cores: the reference's threaded trainer with one memory
        # group (trainer + daemon thread) per two cores, at least one per GPU of
        # the B200 arm, and no more than the mid-stream event window holds
        n_ev = min(cfg["events"], REF_MAX_EVENTS)
        room = (n_ev - int(n_ev * TRAIN_FRAC) // 2) // ((warm + steps) * batch_of(cfg))
        groups = args.ref_groups or max(world, min(16, (os.cpu_count() or 2) // 2, room))
        shape = (1, 1, groups)
    else:  # i- and j-parallel configs: the reference at the B200 arm's own (i, j, k)
        shape = ours
    value, secs, ev, threads, window = reference_time(cfg, shape, steps, warm, log=log)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "events/s",
        "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": 1e3 * secs / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference gen_synthetic, seed 1)",
        "config": {"workload": cfg["workload"],
                   "parallelism": f"(i,j,k)={shape} host threads (the B200 arm: (i,j,k)={ours}, "
                                  f"one trainer per GPU)",
                   "same_parallelism_as_b200_arm": shape == ours,
                   "global_batch": batch_of(cfg) * shape[0] * shape[2], "host_cpus": os.cpu_count(),
                   "window": {"first_event": window[0], "last_event": window[1]}},
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": threads, "kind": "reference",
                         "sample": f"{steps} barriers at (i,j,k)={shape} x {batch_of(cfg)} events, mid-stream window "
                                   f"[{window[0]}, {window[1]}), run_{'training' if threads > 1 else 'sequential'} "
                                   f"(oracle/_ref)"},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if shape != ours:
        # the reference at the B200 arm's own parallelism, for context
        s1 = min(steps, 4)
        v1, secs1, _, thr1, w1 = reference_time(cfg, ours, s1, warm, log=log)
        line["same_parallelism"] = {"value": v1, "unit": "events/s", "cores": thr1,
                                    "parallelism": f"(i,j,k)={ours}", "steps": s1,
                                    "window": {"first_event": w1[0], "last_event": w1[1]}}
    emit(line)
    return 0


# ----------------------------------------------------------------- B200 arm
def _claim_stdout():
    """Routes fd 1 to stderr (NCCL / library banners) and returns a writer for
    the single JSON result line on the original stdout."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    out = os.fdopen(saved, "w")

    def emit(obj):
        out.write(json.dumps(obj) + "\n")
        out.flush()
    return emit


def main():
    emit = _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=200)
    ap.add_argument("--e2e-chunk", type=int, default=4, help="barriers per run.step call in the e2e loop")
    ap.add_argument("--profile-steps", type=int, default=5)
    ap.add_argument("--cpu-baseline-steps", type=int, default=3)
    ap.add_argument("--ref-max-steps", type=int, default=12)
    ap.add_argument("--ref-groups", type=int, default=0,
                    help="reference arm memory groups (0: one per two host cores, >= n_gpus)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1 and args.gpus != 1:
        print(f"warning: --gpus {args.gpus} without torchrun; running 1 rank", file=sys.stderr)

    if args.impl == "reference":
        return reference_arm(args, world, rank, emit)

    import torch
    import torch.distributed as dist

    import paper_2307_07649_b200 as T

    def log(*a):
        if rank == 0:
            print(*a, file=sys.stderr, flush=True)

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    cfg = CONFIGS[args.config]
    t0 = time.time()
    ctx = T.Context(local_rank)
    # gen_synthetic streamed into HBM (bit-identical to the reference stream)
    g = T.TemporalGraph.synthetic(ctx, T.SynthParams(nodes=cfg["nodes"], events=cfg["events"], d_e=cfg["d_e"],
                                                     seed=1))
    ev_src, ev_dst, ev_t = g.events()
    log(f"stream generated into HBM in {time.time() - t0:.1f}s")
    mc = T.ModelConfig(d_e=cfg["d_e"], num_nodes=cfg["nodes"], max_t=float(ev_t[-1]), **model_dims(cfg))
    train_end = int(round(cfg["events"] * TRAIN_FRAC))
    ijk = ijk_of(cfg, world)
    # weak scaling: every memory copy / team sweeps the training range once per
    # rank along the parallel axis, so the barrier count stays ~ constant in N
    tc = T.TrainConfig(i=ijk[0], j=ijk[1], k=ijk[2], local_batch=batch_of(cfg), lr_base=1e-3, seed=1, epochs=world)
    run = T.Run(ctx, g, mc, tc, 0, train_end, rank=rank, nranks=world)
    need = args.warmup + args.steps + 3 * args.profile_steps + args.e2e_steps + 1
    if run.barriers < need:
        raise SystemExit(f"schedule has {run.barriers} barriers, need {need}")
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(T.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        run.comm_init(bytes(uid.cpu().numpy().tobytes()))
    log(f"setup {time.time() - t0:.1f}s; {run.barriers} barriers, {run.nparam} params, (i,j,k)={ijk}")

    launches = run.launches_per_barrier()
    # mid-stream window: fast-forward so the timed barriers are
    # centred on the middle of the schedule, where the CPU reference is timed too
    first_timed = run.barriers // 2 - args.steps // 2
    start = max(0, min(first_timed - args.warmup, run.barriers - need))
    if start > 0:
        run.step(start)
    run.step(args.warmup)
    ctx.synchronize()

    # ---- timed region: K barriers, CUDA events on the context stream
    stream = torch.cuda.ExternalStream(ctx.stream_ptr)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    first = run.next
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        run.step(args.steps)
        e1.record(stream)
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    ctx.synchronize()
    losses = run.losses(first, args.steps)  # also checks the non-finite flag
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    events = run.traversed(first, args.steps)
    value = events / (ms_max / 1e3)
    _, tsched = T.schedule_query(tc, 0, train_end, rank, first, args.steps)
    act = [x for x in range(args.steps) if tsched["active"][x]]
    window = {"first_event": int(min(tsched["slice_begin"][x] for x in act)) if act else None,
              "last_event": int(max(tsched["slice_end"][x] for x in act)) if act else None,
              "barriers": [first, first + args.steps], "of_rank": rank, "schedule_barriers": run.barriers}
    log(f"timed {args.steps} barriers [{first}, {first + args.steps}): {ms_max:.2f} ms, {events} events, "
        f"{value:,.0f} events/s, loss {losses[0]:.4f} -> {losses[-1]:.4f}")

    # ---- phase profile and the per-launch GEMM profile (the kernel roofline)
    prof = []
    for _ in range(args.profile_steps):
        ph, sz = run.profile_barrier(direct=True)
        prof.append((ph, sz))
    gprof = [run.profile_barrier(direct=False)[0] for _ in range(args.profile_steps)] if ijk[1] == 1 else []
    ph_graph = {k: float(np.mean([p[k] for p in gprof])) for k in gprof[0]} if gprof else None
    ph_mean = {k: float(np.mean([p[0][k] for p in prof])) for k in prof[0][0]}
    sz_mean = {k: float(np.mean([p[1][k] for p in prof])) for k in prof[0][1]}
    gemm = [run.gemm_profile() for _ in range(args.profile_steps)]
    g_ms = float(np.mean([x[:, 0].sum() for x in gemm]))
    g_flops = float(np.mean([x[:, 1].sum() for x in gemm]))
    g_bytes = float(np.mean([x[:, 2].sum() for x in gemm]))
    g_launches = int(np.mean([len(x) for x in gemm]))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}
    src = "MEASURED_PEAKS.json (burst)" if "when" in peaks else "B200_PROFILING.md fallback"
    secs = g_ms / 1e3
    t_tensor = g_flops / (peaks["bf16_tflops"] * 1e12)
    t_hbm = g_bytes / (peaks["hbm_gbs"] * 1e9)
    tensor_view = {"achieved": g_flops / secs / 1e12, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                   "executed_bf16x3": 3 * g_flops / secs / 1e12}
    hbm_view = {"achieved": g_bytes / secs / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    bound = "hbm" if t_hbm >= t_tensor else "tensor"
    main_v = hbm_view if bound == "hbm" else tensor_view
    step_direct_ms = max(sum(ph_mean.values()), 1e-9)
    roofline = {"kernel": "tc_gemm_kernel group: every tcgen05 GEMM launch of a barrier (bf16x3, TMA, TMEM), "
                          "the largest share of the barrier's launch list",
                "bound": bound, "achieved": main_v["achieved"], "peak": main_v["peak"], "unit": main_v["unit"],
                "frac": main_v["achieved"] / main_v["peak"], "traffic": roofline_traffic(), "peak_source": src,
                "launches_per_step": g_launches, "flops_per_step": g_flops, "algorithmic_bytes_per_step": g_bytes,
                "flops_per_launch": g_flops / max(g_launches, 1),
                "algorithmic_bytes_per_launch": g_bytes / max(g_launches, 1),
                "launch_ms_avg": g_ms / max(g_launches, 1), "gemm_ms_per_step": g_ms,
                "tensor_view": tensor_view, "hbm_view": hbm_view,
                "share_of_step_direct": g_ms / step_direct_ms,
                "per_launch": [[round(float(v), 6) for v in row] for row in gemm[-1]],
                "per_launch_cols": ["ms", "flops", "bytes", "problems", "max_M", "max_splits"]}
    log("phases (ms): " + ", ".join(f"{k}={v:.3f}" for k, v in ph_mean.items()))
    log(f"plan sizes: {sz_mean}; GEMMs {g_launches} launches {g_ms * 1e3:.1f} us/step "
        f"{tensor_view['achieved']:.1f} TFLOP/s {hbm_view['achieved']:.0f} GB/s")
    rstep = step_roofline(sz_mean, cfg, run.nparam, value / world, peaks)

    # ---- end-to-end through the public API: per step H2D of the step's events
    # (src/dst/t/edge features from pinned host memory) + barrier + D2H loss read
    nb, sched = T.schedule_query(tc, 0, train_end, rank, run.next, args.e2e_steps)
    d_e = cfg["d_e"]
    h2d = 0
    act = [x for x in range(args.e2e_steps) if sched["active"][x]]
    w_lo = min([int(sched["slice_begin"][x]) for x in act], default=0)
    w_hi = max([int(sched["slice_end"][x]) for x in act], default=0)
    # the steps' inputs live in pinned host memory before the timed region
    nw = max(w_hi - w_lo, 1)
    p_src = T.pinned_empty((nw,), np.int32)
    p_dst = T.pinned_empty((nw,), np.int32)
    p_t = T.pinned_empty((nw,), np.float64)
    p_f = T.pinned_empty((nw, max(d_e, 1)), np.float32)[:, :d_e]
    p_src[:w_hi - w_lo] = ev_src[w_lo:w_hi]
    p_dst[:w_hi - w_lo] = ev_dst[w_lo:w_hi]
    p_t[:w_hi - w_lo] = ev_t[w_lo:w_hi]
    if d_e:
        p_f[:w_hi - w_lo] = g.edge_feats(w_lo, w_hi - w_lo)
    p_loss = T.pinned_empty((args.e2e_steps,), np.float64)
    if world > 1:
        dist.barrier()
    ctx.synchronize()
    tw0 = time.perf_counter()
    first_e2e = run.next
    def ingest(x):
        nonlocal_h2d = 0
        if x < args.e2e_steps and sched["active"][x]:
            b0, b1 = int(sched["slice_begin"][x]), int(sched["slice_end"][x])
            n = b1 - b0
            if n > 0:
                o = b0 - w_lo
                g.ingest(b0, p_src[o:o + n], p_dst[o:o + n], p_t[o:o + n], p_f[o:o + n])
                nonlocal_h2d = n * (4 + 4 + 8 + 4 * d_e)
        return nonlocal_h2d

    # per step: H2D of the step's events (copy stream, one step ahead: barrier
    # x plans barrier x + 1, so x + 1's events must be resident before it),
    # the barrier, the D2H of its loss; the host runs ahead, one sync at the
    # end. Barriers are enqueued --e2e-chunk at a time (one graph launch), each
    # with its own ingestion call before and its own loss read after.
    h2d += ingest(0)
    x = 0
    while x < args.e2e_steps:
        c = min(args.e2e_chunk, args.e2e_steps - x)
        for y in range(x + 1, x + c + 1):
            h2d += ingest(y)
        run.step(c)
        for y in range(x, x + c):
            run.loss_async(run.next - c + (y - x), p_loss[y:y + 1])
        x += c
    ctx.synchronize()
    assert np.all(np.isfinite(p_loss))
    e2e_s = time.perf_counter() - tw0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_events = run.traversed(first_e2e, args.e2e_steps)
    e2e_value = e2e_events / float(e2e_t.item())

    # diagnostic: a plain NCCL all-reduce of one flat gradient (no overlap)
    allreduce_us = None
    if world > 1:
        buf = torch.zeros(run.nparam, dtype=torch.float32, device="cuda")
        for _ in range(3):
            dist.all_reduce(buf)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(20):
            dist.all_reduce(buf)
        a1.record()
        a1.synchronize()
        allreduce_us = a0.elapsed_time(a1) * 1e3 / 20

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import ref
        if ref.available():
            v, secs, ev, thr, cw = reference_time(cfg, (1, 1, 1), args.cpu_baseline_steps, 0, log=log)
            cpu = {"value": v, "unit": "events/s", "cores": thr, "kind": "reference",
                   "sample": f"{args.cpu_baseline_steps} barriers x {batch_of(cfg)} events, mid-stream window "
                             f"[{cw[0]}, {cw[1]}), run_sequential of the unmodified reference "
                             f"(oracle/_ref), {secs:.1f}s",
                   "window": {"first_event": cw[0], "last_event": cw[1]}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32 (tcgen05 bf16x3 GEMMs, fp32 accumulate; f64 times)",
            "data": "synthetic (bit-identical gen_synthetic, seed 1)",
            "config": {"workload": cfg["workload"],
                       "parallelism": f"(i,j,k)={ijk}, one trainer per GPU",
                       "global_batch": batch_of(cfg) * ijk[0], "local_batch": batch_of(cfg),
                       "window": window,
                       "l2": "inputs larger than L2 (edge features "
                             f"{cfg['events'] * cfg['d_e'] * 4 / 1e6:.0f} MB; each step reads a new "
                             "event window); no explicit flush"},
            "e2e": {"value": e2e_value, "unit": "events/s",
                    "h2d_bytes_per_step": int(h2d / max(args.e2e_steps, 1)),
                    "d2h_bytes_per_step": 8},
            "gpu_launches": (launches * args.steps) if launches is not None else None,
            "gpu_launches_per_step": launches,
            "roofline": roofline,
            "roofline_step": rstep,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "phases_ms": ph_mean,
            "phases_ms_graph_critical_path": ph_graph,
            "plan_sizes": sz_mean,
            "model_tflops": step_model_flops(sz_mean, cfg) * world / (ms_max / args.steps / 1e3) / 1e12,
            "loss_first_last": [float(losses[0]), float(losses[-1])],
            "grad_allreduce_us_standalone": allreduce_us,
        }
        emit(line)
    run.close()
    g.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
