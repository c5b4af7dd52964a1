#!/usr/bin/env python
"""bench.py — AttnCache hot-path benchmark (BASELINE.json metric: cached-attention prefill
tokens/sec and speedup vs full attention; search QPS).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama32_1b] [--impl ours|reference]

A step is one pass of the whole hot path over one query batch of the
config: search (Alg. 1 l.255-257) -> O = A.V for hits (Alg. 2 l.373-375) -> causal
softmax attention for misses (Alg. 2 l.376-381).  Default workload: BASELINE.json configs[1]
(Llama-3.2-1B-shaped, fits one B200).  Inputs are seeded synthetic (synth/) and resident in
HBM; per-step footprint (~5 GB of maps/V/O) exceeds the 126 MB L2, so no flush is needed.
Prints ONE JSON line on rank 0.

--impl reference times the CPU oracle (oracle/, the only reference this paper-only tier
has) on a bounded sample of the same workload and extrapolates to a full step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "cached-attention prefill tokens/sec"
PAPER_CONTEXT = ("paper (PAPER.md:51, :446, :568; Table 3): 3x attention / 1.6x end-to-end GPU speedup on one "
                 "A100 80GB, Llama-3-3B fp32, MMLU-STEM; 2x / 1.2x on 2x Xeon Silver 4410Y")


_RDEV = None  # device of the torch.distributed reduction tensors (the GPU on NCCL, the CPU on gloo)


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            m = json.load(f)
        return {"hbm_gbs": m["hbm_gbs"], "bf16_tflops": m["bf16_tflops"],
                "bf16_tflops_sustained": m.get("bf16_tflops_sustained", m["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def tri(S):
    return S * (S + 1) // 2


def apply_bytes_per_hit(cfg):
    """Algorithmic HBM bytes of O = A.V for one hit (all L layers, H heads): lower-triangle map
    + V + O."""
    e_m = torch.tensor([], dtype=synth.torch_dtype(cfg.map_dtype)).element_size()
    e_v = torch.tensor([], dtype=synth.torch_dtype(cfg.act_dtype)).element_size()
    return cfg.L * cfg.H * (tri(cfg.S) * e_m + 2 * cfg.S * cfg.d * e_v)


def attend_bytes_per_miss(cfg):
    e_v = torch.tensor([], dtype=synth.torch_dtype(cfg.act_dtype)).element_size()
    return 4 * cfg.L * cfg.H * cfg.S * cfg.d * e_v


def attend_flops_per_miss(cfg):
    """Causal attention flops: 4 d tri(S) per (layer, head)."""
    return 4.0 * cfg.L * cfg.H * cfg.d * cfg.S * (cfg.S + 1) / 2


# ------------------------------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md clocks line)
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index, period_ms=20):
        self.dev = device_index
        self.period_ms = period_ms
        self.proc = None
        self.lines = []
        self.t_mark = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a few hundred ms to start sampling: wait for its first line (at most 3 s) so that the
            # samples cover the timed region that follows (a short region otherwise got 0-1 samples)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self):
        """The timed region starts now: stop() keeps only the samples taken from here on."""
        self.t_mark = time.time()

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = [ln for t, ln in self.lines if self.t_mark is None or t >= self.t_mark]
        if not lines and self.lines:  # a timed region shorter than the sampling period: the sample right after it
            lines = [self.lines[-1][1]]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# ------------------------------------------------------------------------------------------------
def oracle_step_sample(cfg, budget=2.5e9, seed=0):
    """Times the CPU oracle on a bounded sample of one step of `cfg` and extrapolates.

    Each stage gets about `budget` multiply-adds of work (a few seconds of fp64 CPU time on a
    16-core host).  Returns (seconds per full step (extrapolated), description, threads)."""
    import numpy as np
    n_search = int(min(cfg.B, max(4, budget // (cfg.N * cfg.D))))
    n_apply = int(max(4, budget // (cfg.S * cfg.S * cfg.d)))
    n_attend = int(max(4, budget // (cfg.S * cfg.S * cfg.d)))

    import oracle
    from tests._util import storage
    dev = "cpu"
    n_hit = cfg.n_hit
    n_miss = cfg.B - n_hit
    x = synth.features(cfg, 0, cfg.N, dev)
    q, _, _ = synth.queries(cfg, dev)
    rng = np.random.default_rng(seed)
    xs, qs = storage(x), storage(q)
    t0 = time.perf_counter()
    oracle.search(qs[:n_search], xs, cfg.feat_dtype, cfg.tau)
    t_search = (time.perf_counter() - t0) * cfg.B / n_search
    # one entry's maps and one query's V/Q/K provide the sampled (layer, head) units
    maps = storage(synth.maps(cfg, int(rng.integers(cfg.N)), 1, dev))
    V = storage(synth.activations(cfg, "v", 0, 1, device=dev))
    Q = storage(synth.activations(cfg, "q", 0, 1, device=dev))
    K = storage(synth.activations(cfg, "k", 0, 1, device=dev))
    units = cfg.L * cfg.H
    ua = rng.integers(0, units, n_apply)
    t0 = time.perf_counter()
    oracle.apply(maps, cfg.map_dtype, ua * cfg.S * cfg.S, V, cfg.act_dtype, ua * cfg.S * cfg.d, cfg.S, cfg.d)
    t_apply = (time.perf_counter() - t0) * (n_hit * units) / n_apply
    um = rng.integers(0, units, n_attend)
    t0 = time.perf_counter()
    oracle.attend(Q, K, V, cfg.act_dtype, um * cfg.S * cfg.d, cfg.S, cfg.d)
    t_attend = (time.perf_counter() - t0) * (n_miss * units) / n_attend
    desc = (f"extrapolated from {n_search} of {cfg.B} queries' search, {n_apply} of {n_hit * units} hit "
            f"(layer,head) A.V units, {n_attend} of {n_miss * units} miss attention units")
    return t_search + t_apply + t_attend, desc, oracle.get_threads()


def _line_config(cfg, n_hit=None, **extra):
    """The full workload description carried by every line (ours and the reference arm)."""
    d = {"workload": cfg.name, "bj_config_index": cfg.bj_index, "N": cfg.N, "D": cfg.D, "L": cfg.L, "H": cfg.H,
         "S": cfg.S, "d": cfg.d, "B": cfg.B, "tau": cfg.tau, "planted_hit_rate": cfg.hit_rate, "seed": cfg.seed,
         "feat_dtype": cfg.feat_dtype, "map_dtype": cfg.map_dtype, "act_dtype": cfg.act_dtype}
    if n_hit is not None:
        d["hits"] = n_hit
    d.update(extra)
    return d


def run_reference(args, cfg):
    """The reference arm of this paper-only tier: the CPU oracle (oracle/) timed as it stands on the host
    cores, each step a bounded sample of one step of the workload, extrapolated to the full step (so the
    line's ms_per_step is an extrapolation, flagged, while the wall time of the run stays a few minutes)."""
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    import oracle
    oracle.set_threads(os.cpu_count() or 1)
    times, walls = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        t, desc, cores = oracle_step_sample(cfg, seed=i)
        if i >= args.warmup:
            times.append(t)
            walls.append(time.perf_counter() - t0)
    t = statistics.median(times)
    value = cfg.B * cfg.S / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (synth/, seed 0)",
            "extrapolated": True, "sample_wall_s_per_step": statistics.median(walls),
            "config": _line_config(cfg, cfg.n_hit, parallelism="CPU oracle (OpenMP over independent units)"),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------
def run_ours(args, cfg):
    rank, world, local = _env_rank()
    if world > 1 or args.force_dist:
        return run_dist(args, cfg)
    import paper_2510_25979_b200 as ac
    from paper_2510_25979_b200.pipeline import PrefillStep
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = ac.Context(local)
    peaks = _peaks()

    # ---- inputs resident in HBM (untimed) ----
    x = synth.features(cfg, 0, cfg.N, dev)
    # DB building (Fig. 4 step 3): the generator's dense maps are stored in the PACKED layout
    maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), cfg.N, cfg.L, cfg.H, cfg.S,
                           synth.torch_dtype(cfg.map_dtype), dev, chunk=max(1, (1 << 30) // cfg.map_bytes_per_entry))
    db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
    q, _, _ = synth.queries(cfg, dev)
    Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=dev) for k in "qkv")
    O = torch.empty_like(V)
    step = PrefillStep(ctx, db, cfg.tau)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        step(q, Q, K, V, O)
    ctx.sync()
    idx, score, hit = step.search(q)
    n_hit = int(hit.sum().item())

    # ---- timed region: K whole steps, per-stage events on the launch stream ----
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()  # returns once nvidia-smi samples; two more untimed steps re-warm the GPU after that wait
    for _ in range(2):
        step(q, Q, K, V, O)
    torch.cuda.synchronize()
    launches0 = ac.attncache_launch_count()
    clocks.mark()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(args.steps):
        e = ev[k]
        e[0].record(stream)
        idx, score, hit = step.search(q)
        e[1].record(stream)
        ac.attncache_apply_cached(db, idx, V, O, hit=hit)
        e[2].record(stream)
        ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)
        e[3].record(stream)
    end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = ac.attncache_launch_count() - launches0
    ctx.sync()
    total_ms = start.elapsed_time(end)
    ms = total_ms / args.steps
    search_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    apply_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)
    attend_ms = statistics.mean(e[2].elapsed_time(e[3]) for e in ev)

    # ---- comparison: full attention on every row (the paper's "full model" baseline) ----
    O_full = torch.empty_like(V)
    hit_rows_only = (1 - hit).contiguous()
    for _ in range(2):
        ac.attncache_attend_full(ctx, Q, K, V, O_full)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(args.steps):
        ac.attncache_attend_full(ctx, Q, K, V, O_full)
    s1.record(stream)
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for _ in range(args.steps):
        ac.attncache_attend_full(ctx, Q, K, V, O_full, skip=hit_rows_only)
    h1.record(stream)
    torch.cuda.synchronize()
    full_ms = s0.elapsed_time(s1) / args.steps
    full_hits_ms = h0.elapsed_time(h1) / args.steps

    # ---- e2e: the same step through the public API from pinned host buffers ----
    e2e = run_e2e(args, cfg, ctx, db, step, q, Q, K, V, dev, stream)

    # ---- roofline of the dominant kernel (apply_cached) ----
    bytes_alg = n_hit * apply_bytes_per_hit(cfg)
    achieved = bytes_alg / (apply_ms * 1e-3) / 1e9
    traffic = _ncu_traffic(cfg.name, "apply")
    roofline = {"kernel": f"attncache apply_cached ({ac.attncache_variant('apply', V.dtype, cfg.S, cfg.d)})",
                "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "peak_source": f"{peaks['source']} MEASURED_PEAKS.json hbm_gbs",
                "algorithmic_bytes_per_launch": bytes_alg, "avg_launch_ms": apply_ms,
                "note": "launch time measured with CUDA events around the apply_cached call on the launch stream "
                        "inside the timed region (one A.V kernel that selects its rows in its prologue; larger "
                        "batches add a select launch)"}
    attend_alg = (cfg.B - n_hit) * attend_bytes_per_miss(cfg)
    secondary = {
        "search": {"ms": search_ms, "qps": cfg.B / (search_ms * 1e-3),
                   "variant": ac.attncache_variant("search", q.dtype, 0, cfg.D)},
        "attend_full_misses": {"ms": attend_ms, "hbm_frac": attend_alg / (attend_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                               "tensor_frac": (cfg.B - n_hit) * attend_flops_per_miss(cfg) / (attend_ms * 1e-3) / 1e12
                               / peaks["bf16_tflops"],
                               "variant": ac.attncache_variant("attend", V.dtype, cfg.S, cfg.d)},
    }

    line = {"metric": METRIC, "value": cfg.B * cfg.S / (ms * 1e-3), "unit": "tokens/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": cfg.act_dtype, "data": "synthetic (synth/, seed 0)",
            "config": _line_config(cfg, n_hit, parallelism="single GPU", l2="inputs exceed L2 (no flush)"),
            "warmup_steps_run": args.warmup + 2,
            "speedup_vs_full_attention": {"batch": full_ms / ms, "per_hit_kernel": full_hits_ms / apply_ms,
                                          "full_attention_ms": full_ms, "paper_context": PAPER_CONTEXT},
            "search_qps": cfg.B / (search_ms * 1e-3),
            "stages": secondary, "roofline": roofline, "e2e": e2e, "gpu_launches": launches, "clocks": clk}
    # §8(f) f1, DB building: capture the misses' maps (Q, K -> packed bf16 DB entries)
    secondary["capture_misses"] = capture_stage(ac, ctx, cfg, Q, K, hit, stream, max(3, args.steps), peaks)
    # small batches (a serving request at a time): per-step time eager vs one CUDA-graph replay
    secondary["small_batch"] = small_batch_stage(ac, ctx, db, cfg, q, Q, K, V, stream)
    # §8(f) f2: the feature projector (Alg. 1 l.254) on this batch and at a tensor-bound batch
    secondary["project"] = project_stage(ac, ctx, cfg, dev, stream, max(3, args.steps), peaks)
    # paper-comparable baseline: eager torch attention (matmul -> masked softmax -> matmul, the
    # unfused attention of PAPER.md Table 4's "AM" + "AM.V" rows) on every row of the batch
    eager_ms = eager_attention_ms(Q, K, V, stream, max(2, args.steps // 2))
    line["speedup_vs_full_attention"]["eager_torch_attention_ms"] = eager_ms
    line["speedup_vs_full_attention"]["batch_vs_eager_torch"] = eager_ms / ms
    del O_full
    # §8(f) f4: Eq. 5 block level (Q/K/V projections + RoPE + attention vs V projection + A.V)
    line["eq5_block"] = eq5_block(ac, ctx, db, cfg, idx, hit, stream, max(3, args.steps // 2))
    if cfg.H % 8 == 0:
        line["eq5_block_gqa"] = eq5_block(ac, ctx, db, cfg, idx, hit, stream, max(3, args.steps // 2), n_kv_heads=8)
    if not args.no_target and cfg.name != "llama3_8b":
        # north_star's target shape (>= 3x at Llama-3-8B shape: BASELINE.json configs[2], Table 4)
        del step, db, maps, x, q, Q, K, V, O, idx, score, hit, hit_rows_only
        torch.cuda.empty_cache()
        line["north_star_target"] = target_config_block(args, ac, ctx, dev, stream, peaks, "llama3_8b")
    if not args.no_search_sweep:
        line["search_sweep"] = search_sweep(ac, ctx, dev, stream, max(3, args.steps), peaks)
    if not args.no_cpu_baseline:
        import oracle
        oracle.set_threads(os.cpu_count() or 1)
        t, desc, cores = oracle_step_sample(cfg)
        oracle.set_threads(1)  # BASELINE.md's CPU plan: also at one thread (a smaller sample)
        t1, desc1, _ = oracle_step_sample(cfg, budget=6e8)
        oracle.set_threads(os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": cfg.B * cfg.S / t, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                                "sample": desc, "extrapolated": True,
                                "one_thread": {"value": cfg.B * cfg.S / t1, "unit": "tokens/s", "cores": 1,
                                               "sample": desc1}}
    print(json.dumps(line), flush=True)
    return 0


def target_config_block(args, ac, ctx, dev, stream, peaks, name):
    """The whole step at another BASELINE.json config (default: configs[2], Llama-3-8B shape, where north_star
    states its >= 3x target): step time and tokens/s, per-stage times, the A.V and attention rooflines, the
    speedups over in-library full attention (batch and per hit), and the Eq. 5 block ratio."""
    from paper_2510_25979_b200.pipeline import PrefillStep
    cfg = synth.CONFIGS[name]
    x = synth.features(cfg, 0, cfg.N, dev)
    maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), cfg.N, cfg.L, cfg.H, cfg.S,
                           synth.torch_dtype(cfg.map_dtype), dev, chunk=max(1, (1 << 30) // cfg.map_bytes_per_entry))
    db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
    q, _, _ = synth.queries(cfg, dev)
    Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=dev) for k in "qkv")
    O = torch.empty_like(V)
    step = PrefillStep(ctx, db, cfg.tau)
    steps = max(3, min(args.steps, 20))
    for _ in range(max(3, args.warmup)):
        step(q, Q, K, V, O)
    ctx.sync()
    idx, score, hit = step.search(q)
    n_hit = int(hit.sum().item())
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    for k in range(steps):
        e = ev[k]
        e[0].record(stream)
        step.search(q)
        e[1].record(stream)
        ac.attncache_apply_cached(db, idx, V, O, hit=hit)
        e[2].record(stream)
        ac.attncache_attend_full(ctx, Q, K, V, O, skip=hit)
        e[3].record(stream)
    torch.cuda.synchronize()
    search_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    apply_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)
    attend_ms = statistics.mean(e[2].elapsed_time(e[3]) for e in ev)
    ms = statistics.mean(e[0].elapsed_time(e[3]) for e in ev)

    def timed(fn):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    O_full = torch.empty_like(V)
    full_ms = timed(lambda: ac.attncache_attend_full(ctx, Q, K, V, O_full))
    miss_rows = (1 - hit).contiguous()
    full_hits_ms = timed(lambda: ac.attncache_attend_full(ctx, Q, K, V, O_full, skip=miss_rows))
    del O_full
    bytes_alg = n_hit * apply_bytes_per_hit(cfg)
    attend_alg = (cfg.B - n_hit) * attend_bytes_per_miss(cfg)
    out = {"workload": cfg.name, "bj_config_index": cfg.bj_index, "config": _line_config(cfg, n_hit),
           "ms_per_step": ms, "tokens_per_s": cfg.B * cfg.S / (ms * 1e-3), "steps": steps,
           "stages_ms": {"search": search_ms, "apply_cached": apply_ms, "attend_full_misses": attend_ms},
           "apply_roofline": {"bound": "hbm", "achieved": bytes_alg / (apply_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
                              "unit": "GB/s", "frac": bytes_alg / (apply_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                              "algorithmic_bytes_per_launch": bytes_alg,
                              "traffic": _ncu_traffic(cfg.name, "apply")},
           "attend_misses_hbm_frac": attend_alg / (attend_ms * 1e-3) / 1e9 / peaks["hbm_gbs"] if attend_ms else None,
           "speedup_vs_full_attention": {"batch": full_ms / ms, "per_hit_kernel": full_hits_ms / apply_ms,
                                         "full_attention_ms": full_ms, "full_attention_hit_rows_ms": full_hits_ms,
                                         "ceiling_vs_roofline_attention_per_hit": 8 * cfg.d / (cfg.S + 1 + 4 * cfg.d),
                                         "paper_context": PAPER_CONTEXT},
           "eq5_block": eq5_block(ac, ctx, db, cfg, idx, hit, stream, steps),
           "eq5_block_gqa": eq5_block(ac, ctx, db, cfg, idx, hit, stream, steps, n_kv_heads=8)}
    del step, db, maps, x, q, Q, K, V, O
    torch.cuda.empty_cache()
    return out


def capture_stage(ac, ctx, cfg, Q, K, hit, stream, steps, peaks):
    """DB building (f1): maps of the batch's misses written as PACKED DB entries; HBM roofline on
    Q + K read and the packed maps written."""
    P = ac.attncache_packed_map_elems(cfg.S)
    out = torch.empty(cfg.B, cfg.L, cfg.H, P, dtype=synth.torch_dtype(cfg.map_dtype), device=Q.device)
    ac.attncache_capture_maps(ctx, Q, K, map_dtype=out.dtype, packed=True, out=out, skip=hit)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        ac.attncache_capture_maps(ctx, Q, K, map_dtype=out.dtype, packed=True, out=out, skip=hit)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    n_miss = int((hit == 0).sum().item())
    nbytes = n_miss * cfg.L * cfg.H * (2 * cfg.S * cfg.d * Q.element_size() + P * out.element_size())
    del out
    return {"ms": ms, "bytes": nbytes, "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
            "variant": ac.attncache_variant("capture", Q.dtype, cfg.S, cfg.d)}


def small_batch_stage(ac, ctx, db, cfg, q, Q, K, V, stream, iters=50):
    """Latency-bound batches of B = 1 and 8 prefills (the first rows of the batch): the whole step issued
    eagerly (six library launches plus host-side checks per step) vs replayed as one CUDA graph
    (pipeline.GraphedPrefillStep)."""
    from paper_2510_25979_b200.pipeline import GraphedPrefillStep, PrefillStep
    step = PrefillStep(ctx, db, cfg.tau)
    out = []
    for B in (1, 8):
        qb, Qb, Kb, Vb = (t[:B].contiguous() for t in (q, Q, K, V))
        Ob = torch.empty_like(Vb)
        g = GraphedPrefillStep(step, qb, Qb, Kb, Vb)

        def timed(fn):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(iters):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / iters

        eager = timed(lambda: step(qb, Qb, Kb, Vb, Ob))
        graph = timed(g.replay)
        out.append({"B": B, "eager_ms": eager, "graph_ms": graph, "graph_tokens_per_s": B * cfg.S / (graph * 1e-3)})
        del g
    return out


def project_stage(ac, ctx, cfg, dev, stream, steps, peaks):
    """f2, Alg. 1 l.254: f = normalize(W2 relu(W1 h + b1) + b2) (synthetic weights, reading R31) at the config's
    batch and at B = 8192 (tensor-bound); roofline on flops 2B(E*Hd + Hd*D) vs bytes (weights + h + f)."""
    out = []
    for B in (cfg.B, 8192):
        h, W1, b1, W2, b2 = synth.projector_inputs(cfg, B=B, device=dev)
        f = torch.empty(B, cfg.D, dtype=synth.torch_dtype(cfg.feat_dtype), device=dev)
        ac.attncache_project_features(ctx, h, W1, b1, W2, b2, out=f)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            ac.attncache_project_features(ctx, h, W1, b1, W2, b2, out=f)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        E, Hd, D = h.shape[1], W1.shape[0], cfg.D
        flops = 2.0 * B * (E * Hd + Hd * D)
        nbytes = (Hd * E + D * Hd) * h.element_size() + B * E * h.element_size() + B * D * f.element_size()
        out.append({"B": B, "E": E, "hidden": Hd, "D": D, "ms": ms, "tflops": flops / (ms * 1e-3) / 1e12,
                    "tensor_frac": flops / (ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
                    "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                    "variant": ac.attncache_variant("project", h.dtype, E, Hd)})
        del h, W1, W2, f
    return out


def eq5_block(ac, ctx, db, cfg, idx, hit, stream, steps, n_kv_heads=None):
    """One layer's attention block for the whole batch: the full path on every row vs the cached
    path (hits: V projection + A.V; misses: the full path), and the all-hit per-row ratio.  The paper's
    3x attention speedup is this block-level quantity (Table 4).  n_kv_heads: grouped-query
    K / V projections (a supplementary variant; the configs are multi-head, reading A14)."""
    from paper_2510_25979_b200.block import AttentionBlock
    X, (Wq, Wk, Wv) = synth.block_inputs(cfg, idx.device, n_kv_heads=n_kv_heads)
    blk = AttentionBlock(ctx, db, Wq, Wk, Wv, cfg.H, cfg.d, layer=0)
    miss_rows = torch.nonzero(hit == 0).flatten()
    none = miss_rows[:0]
    all_hit = torch.ones_like(hit)

    def timed(fn):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    full_ms = timed(lambda: blk.full(X))
    cached_ms = timed(lambda: blk.cached(X, idx, hit, miss_rows))
    hits_ms = timed(lambda: blk.cached(X, idx, all_hit, none))
    del X, Wq, Wk, Wv, blk
    out = {"layer_full_ms": full_ms, "layer_cached_ms": cached_ms, "layer_all_hits_ms": hits_ms,
           "speedup_batch": full_ms / cached_ms, "speedup_per_hit": full_ms / hits_ms,
           "note": "one layer, whole batch; Q/K/V projections (attncache_linear), RoPE, A.V and attention all "
                   "in this library; synthetic weights; paper: 3x attention on A100 (PAPER.md:446)"}
    if n_kv_heads is not None:
        out["n_kv_heads"] = n_kv_heads
        out["note"] += (f"; grouped-query variant: W_K, W_V with {n_kv_heads} KV heads (the Llama-3 count), "
                        "maps and A.V per query head")
    return out


def eager_attention_ms(Q, K, V, stream, steps):
    """Unfused torch attention (a comparison point, not this library's path)."""
    S = Q.shape[-2]
    mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=Q.device), diagonal=1)
    scale = 1.0 / math.sqrt(Q.shape[-1])

    B = Q.shape[0]
    per_row = Q[0].numel() // Q.shape[-1] * S * 4  # fp32 score bytes of one batch row
    rows = max(1, min(B, (8 << 30) // per_row))    # bound the materialised scores to ~8 GB

    def run():
        for b0 in range(0, B, rows):
            q, k, v = Q[b0:b0 + rows], K[b0:b0 + rows], V[b0:b0 + rows]
            s = torch.matmul(q, k.transpose(-1, -2)) * scale
            s.masked_fill_(mask, float("-inf"))
            torch.matmul(torch.softmax(s, dim=-1, dtype=torch.float32).to(v.dtype), v)

    run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def search_sweep(ac, ctx, dev, stream, steps, peaks):
    """BASELINE.json configs[4]: exact top-1 over 1M x 1024 bf16 features at B = 1/64/1024/8192
    (half planted hits); search QPS and roofline fractions (K1 + K2)."""
    cfg = synth.CONFIGS["search_sweep"]
    x = synth.features(cfg, 0, cfg.N, dev)
    db = ac.Database(ctx, x)
    out = {"workload": "search_sweep (BASELINE.json configs[4])", "N": cfg.N, "D": cfg.D, "points": []}
    for B in (1, 64, 1024, 8192):
        q, pos, _ = synth.queries(cfg, dev, B=B)
        idx, score, hit = ac.attncache_search(db, q, cfg.tau)
        for _ in range(2):
            ac.attncache_search(db, q, cfg.tau, idx, score, hit)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            ac.attncache_search(db, q, cfg.tau, idx, score, hit)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        nbytes = (cfg.N + B) * cfg.D * 2 + 8 * B
        flops = 2.0 * B * cfg.N * cfg.D
        out["points"].append({"B": B, "ms": ms, "qps": B / (ms * 1e-3), "hits": int(hit.sum().item()),
                              "planted_hits": len(pos),
                              "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                              "tensor_frac": flops / (ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
                              "tensor_frac_sustained": flops / (ms * 1e-3) / 1e12 / peaks["bf16_tflops_sustained"],
                              "variant": ac.attncache_variant("search", q.dtype, 0, cfg.D)})
    del db, x
    return out


def _rows_activations(cfg, kind, rows, dev):
    """Q/K/V of the given global query positions (the same seeds as synth.activations)."""
    out = torch.empty(len(rows), cfg.L, cfg.H, cfg.S, cfg.d, dtype=synth.torch_dtype(cfg.act_dtype), device=dev)
    for k, b in enumerate(rows):
        synth.activations(cfg, kind, b, 1, out=out[k:k + 1])
    return out


def _dist_timed(args, cfg, ac, ctx, db, dev, placement, world, rank, local):
    """Builds one rank's inputs for the global batch cfg.B (home blocks: contiguous, shard_range) and times
    K steps of the chosen placement; returns (ms max over ranks, extra dict, launches, hits)."""
    import torch.distributed as dist

    from paper_2510_25979_b200.dist import AffinityPrefill, ShardedPrefill, shard_range
    q_all, _, _ = synth.queries(cfg, dev)
    hb, hc = shard_range(cfg.B, world, rank)
    q = q_all[hb:hb + hc].contiguous()
    sizes = [shard_range(cfg.B, world, r)[1] for r in range(world)]
    comp = torch.cuda.current_stream(dev)
    if placement == "affinity":
        step = AffinityPrefill(ctx, db, cfg.tau, sizes, hit_cost=apply_bytes_per_hit(cfg),
                               miss_cost=attend_bytes_per_miss(cfg))
        plan0 = step.plan(q)
        loc = step.local_queries(plan0)
        # the synthetic activations of the queries this rank processes, generated here from their seeds
        # (in a model they come from the relocated hidden states)
        Q, K, V = (_rows_activations(cfg, k, loc.tolist(), dev) for k in "qkv")
        O = torch.empty_like(V)
        X_home = torch.randn(hc, cfg.S, cfg.H * cfg.d, device=dev).to(synth.torch_dtype(cfg.act_dtype))
        # side streams at high priority: when a persistent layer kernel's CTAs retire, the block scheduler
        # dispatches the next batch's search / placement / copy CTAs before the next layer kernel's
        side_prio = int(os.environ.get("ATTNCACHE_BENCH_SIDE_PRIORITY", "-1"))
        comm, plan_st = torch.cuda.Stream(dev, priority=side_prio), torch.cuda.Stream(dev, priority=side_prio)
        state = {"plan": plan0}
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        budget = (sms - args.aux_sms, args.aux_sms) if 0 < args.aux_sms < sms else (sms, sms)
        # the layers' persistent kernels leave aux_sms SMs to the next batch's search, placement, relocation
        # copies and NCCL kernels on the side streams (attncache_ctx_set_sm_budget)
        ctx.set_sm_budget(*budget)

        def one_step():
            # steady state of a serving loop: this batch's layers run locally on the compute stream (planned and
            # relocated during the previous step), while the NEXT batch's sharded search and placement (plan
            # stream; its one host round trip for the send/recv counts stalls only that stream) and the
            # relocation of its request state (communication stream) run beside them.  The bench repeats one
            # batch, so every step does one batch's search, placement, relocation and layers; the step ends when
            # all three streams are done.
            cur = state["plan"]
            if state.get("timing") is not None:  # events around the local A.V (the line's roofline kernel)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(comp)
                step.apply_local(cur, loc, V, O)
                e1.record(comp)
                state["timing"].append((e0, e1))
                if loc.numel():
                    ac.attncache_attend_full(ctx, Q, K, V, O, skip=cur["hit_loc"])
            else:
                step.apply_local(cur, loc, V, O, Q, K)
            for t in (cur["idx_loc"], cur["hit_loc"]):  # made on the plan stream, read here (caching allocator)
                t.record_stream(comp)
            nxt = step.plan(q, stream=plan_st)
            comm.wait_stream(plan_st)
            step.relocate(X_home, nxt, stream=comm)
            nxt["send_order"].record_stream(comm)
            comp.wait_stream(comm)
            state["plan"] = nxt
            return nxt
    else:
        Q, K, V = (synth.activations(cfg, k, hb, hc, device=dev) for k in "qkv")
        O = torch.empty_like(V)
        step = ShardedPrefill(ctx, db, cfg.tau, sizes)
        one_step = lambda: step(q, Q, K, V, O)  # noqa: E731
    # at least 10 untimed steps: with 3 the first timed run of the pipelined step was 5-8 % slower in about half the
    # runs (its side streams' first allocations and NCCL's lazy setup still settling), with 10 within 1.5 %
    for _ in range(max(args.warmup, 10)):
        res = one_step()
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = ac.attncache_launch_count()
    if placement == "affinity":
        state["timing"] = []
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(comp)
    for _ in range(args.steps):
        res = one_step()
    end.record(comp)
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([start.elapsed_time(end) / args.steps], device=_RDEV)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)  # the step time is the slowest rank's
    launches = torch.tensor([ac.attncache_launch_count() - launches0], device=_RDEV)
    dist.all_reduce(launches)
    extra = {}
    if placement == "affinity":
        assert torch.equal(step.local_queries(res), loc), "placement changed between steps"
        n_hit = int(res["hit"].sum().item())
        per_rank = torch.tensor([loc.numel()], device=_RDEV)
        gathered = [torch.empty_like(per_rank) for _ in range(world)]
        dist.all_gather(gathered, per_rank)
        av_ms = sum(a.elapsed_time(b) for a, b in state["timing"]) / max(1, len(state["timing"]))
        n_hit_loc = int(res["hit_loc"].sum().item()) if loc.numel() else 0
        extra = {"_av": (av_ms, n_hit_loc * apply_bytes_per_hit(cfg)),
                 "sm_budget": {"compute_sms": budget[0], "aux_sms": budget[1]},
                 "queries_per_rank": [int(t.item()) for t in gathered],
                 "plan_load_bytes_per_rank": [float(v) for v in res["load"].tolist()],
                 "relocated_bytes_per_query": cfg.S * cfg.H * cfg.d * 2,
                 "pipelining": "the next batch's search + placement (plan stream) and request-state relocation "
                               "(attncache_relocate_rows, communication stream) overlap this batch's local A.V / "
                               "attention; all complete inside the step"}
    else:
        t = torch.tensor([int(res[2].sum().item())], device=_RDEV)
        dist.all_reduce(t)
        n_hit = int(t.item())
    del Q, K, V, O
    return float(ms.item()), extra, int(launches.item()), n_hit


def _dist_e2e(args, cfg, ctx, db, dev, world, rank):
    """The N > 1 end-to-end leg: each rank's home block of the batch from PINNED host memory through the
    library's collective calls (dist.ShardedPrefill's search, then the routed A.V and the local attention), with
    every host <-> device copy inside the timed region: H2D of the home queries and V, the decisions to the host
    (one sync: only the misses' Q and K cross the host link, Alg. 2 l.376-378), H2D of those Q / K rows, then
    D2H of O.  Routed placement (the request state never moves).  Wall clock of K steps, max over ranks."""
    import torch.distributed as dist

    from paper_2510_25979_b200.dist import ShardedPrefill, shard_range
    import paper_2510_25979_b200 as ac
    q_all, _, _ = synth.queries(cfg, dev)
    hb, hc = shard_range(cfg.B, world, rank)
    sizes = [shard_range(cfg.B, world, r)[1] for r in range(world)]
    step = ShardedPrefill(ctx, db, cfg.tau, sizes)
    qh = q_all[hb:hb + hc].contiguous().cpu().pin_memory()
    Qh, Kh, Vh = (synth.activations(cfg, k, hb, hc, device=dev).cpu().pin_memory() for k in "qkv")
    # O double-buffered: step i's D2H of O runs on a copy stream beside step i + 1's H2D and kernels
    Ohs = [torch.empty(Vh.shape, dtype=Vh.dtype).pin_memory() for _ in range(2)]
    dq, dQ, dK, dV = (torch.empty(t.shape, dtype=t.dtype, device=dev) for t in (qh, Qh, Kh, Vh))
    dOs = [torch.empty_like(dV) for _ in range(2)]
    comp, cs = torch.cuda.current_stream(dev), torch.cuda.Stream(dev)
    out_done = [torch.cuda.Event(), torch.cuda.Event()]
    row = Vh[0].numel() * Vh.element_size() if hc else 0
    n_miss = [0]

    def one(i):
        dO, Oh = dOs[i % 2], Ohs[i % 2]
        dq.copy_(qh, non_blocking=True)
        dV.copy_(Vh, non_blocking=True)
        idx, score, hit = step.search(dq)
        miss = torch.nonzero(hit == 0).flatten().cpu()  # the decisions to the host (one sync of this stream)
        n_miss[0] = miss.numel()
        for m in miss.tolist():  # only the misses' Q and K cross the host link
            dQ[m].copy_(Qh[m], non_blocking=True)
            dK[m].copy_(Kh[m], non_blocking=True)
        comp.wait_event(out_done[i % 2])  # the D2H of step i - 2 has read this O buffer
        step.apply_routed(idx, hit, dV, dO)
        if miss.numel():
            ac.attncache_attend_full(ctx, dQ, dK, dV, dO, skip=hit)
        cs.wait_stream(comp)
        with torch.cuda.stream(cs):
            Oh.copy_(dO, non_blocking=True)
            out_done[i % 2].record(cs)

    for i in range(max(1, args.warmup)):
        one(i)
    torch.cuda.synchronize()
    dist.barrier()
    n = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for i in range(n):
        one(i)
    torch.cuda.synchronize()  # the last step's O is in host memory
    ms = torch.tensor([(time.perf_counter() - t0) * 1e3 / n], device=_RDEV)
    dist.barrier()
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    h2d = torch.tensor([qh.numel() * qh.element_size() + Vh.numel() * Vh.element_size() + 2 * n_miss[0] * row],
                       device=_RDEV, dtype=torch.float64)
    d2h = torch.tensor([Ohs[0].numel() * Ohs[0].element_size() + hc * 13], device=_RDEV, dtype=torch.float64)
    dist.all_reduce(h2d)
    dist.all_reduce(d2h)
    return {"value": cfg.B * cfg.S / (float(ms.item()) * 1e-3), "unit": "tokens/s", "ms_per_step": float(ms.item()),
            "steps": n, "h2d_bytes_per_step": int(h2d.item()), "d2h_bytes_per_step": int(d2h.item()),
            "api": "dist.ShardedPrefill (attncache_search / attncache_apply_cached COLLECTIVE, attncache_attend_full)",
            "note": "pinned host buffers per rank, routed placement, global batch of the line's B (bytes summed "
                    "over ranks); O double-buffered so a step's D2H overlaps the next step's H2D; wall clock of K "
                    "steps ending when the last O is in host memory, max over ranks"}


def run_dist(args, cfg):
    """N > 1 (torchrun, one process per GPU): the DB is sharded by contiguous entry ranges over the GPUs and
    every exchange runs inside libattncache over its own NCCL communicator (torch.distributed only
    broadcasts the NCCL unique id and provides the barrier / max-over-ranks timing).  Each rank is home to a
    contiguous block of the query batch.  Measured both ways:
      weak   : the config's batch on EVERY GPU (global batch B * N against the same sharded DB);
      strong : the config's batch split over the GPUs (the same global data at every N; SURVEY.md:737).
    `--scaling` picks which one is the line's value; the other is reported beside it.
      --placement affinity (default; SURVEY.md §8(e) owner-affinity): search_all, the device placement, one
        relocation of the request state, then A.V / attention locally;
      --placement routed (the north_star's literal routing): hits' V rows go to the owner and O rows come back
        inside attncache_apply_cached, misses stay home."""
    import torch.distributed as dist

    import paper_2510_25979_b200 as ac
    from paper_2510_25979_b200.dist import shard_range
    if "MASTER_ADDR" not in os.environ:  # --force-dist without torchrun: a one-rank group
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]), RANK="0",
                              WORLD_SIZE="1", LOCAL_RANK="0")
    rank, world, local = _env_rank()
    global _RDEV
    if os.environ.get("ATTNCACHE_TEST_SINGLE_DEVICE") == "1":
        # functional test of the N > 1 path on one GPU (tests/test_gpu_fake_nccl.py): every rank on GPU 0, the
        # library's NCCL calls in tests/native/fake_nccl.cpp, torch.distributed on gloo; its times mean nothing
        local = 0
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        dist.init_process_group("gloo")
        _RDEV = torch.device("cpu")
    else:
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        dist.init_process_group("nccl", device_id=dev)
        _RDEV = dev
    ctx = ac.Context.from_process_group(local)  # the library's own NCCL communicator
    begin, count = shard_range(cfg.N, world, rank)
    x = synth.features(cfg, begin, count, dev)
    maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, begin + b), count, cfg.L, cfg.H, cfg.S,
                           synth.torch_dtype(cfg.map_dtype), dev, chunk=max(1, (1 << 30) // cfg.map_bytes_per_entry))
    db = ac.Database(ctx, x, maps, n_global=cfg.N, shard_begin=begin, packed=True, seq_len=cfg.S)  # collective
    # a slower sampling period here: the pipelined step has host round trips, and NVML queries every 20 ms
    # measurably slowed it (world-1: 1.16-1.19 against 1.10-1.11 ms)
    clocks = ClockSampler(local, period_ms=200)
    clocks.start()
    clocks.mark()  # the warm-up and timed steps of both runs follow
    runs = {}
    for mode in (args.scaling, "strong" if args.scaling == "weak" else "weak"):
        c = cfg.with_(B=cfg.B * world) if mode == "weak" else cfg
        runs[mode] = (c,) + _dist_timed(args, c, ac, ctx, db, dev, args.placement, world, rank, local)
    clk = clocks.stop()
    e2e_cfg = runs[args.scaling][0]
    e2e = _dist_e2e(args, e2e_cfg, ctx, db, dev, world, rank)
    ctx.sync()
    if rank == 0:
        c, ms, extra, launches, n_hit = runs[args.scaling]
        oc, oms, oextra, _, on_hit = runs["strong" if args.scaling == "weak" else "weak"]
        par = (f"DB sharded by entry over {world} GPUs; collectives inside libattncache (NCCL); " +
               ("owner-affinity placement: hits on the owner, misses on the least-loaded GPUs, request state "
                "moved once, all layers local" if args.placement == "affinity" else
                "hits routed to the owner (V out, O back by grouped NCCL send/recv inside apply_cached)"))
        av = extra.pop("_av", None)
        oextra.pop("_av", None)
        if av and av[0] > 0 and av[1] > 0:
            ach = av[1] / (av[0] * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": _peaks()["hbm_gbs"], "unit": "GB/s",
                    "frac": ach / _peaks()["hbm_gbs"], "traffic": None,
                    "note": "rank 0's local A.V (attncache_apply_cached_local): its hits' algorithmic bytes / the "
                            "launch's average CUDA-event duration on the compute stream, inside the timed steps; "
                            "peak per GPU"}
        else:
            roof = {"bound": "hbm", "achieved": None, "peak": _peaks()["hbm_gbs"], "unit": "GB/s", "frac": None,
                    "traffic": None, "note": "routed placement (the A.V call includes the exchanges) or no local "
                                             "hit on rank 0: the per-kernel roofline is the N = 1 run's"}
        line = {"metric": METRIC, "value": c.B * c.S / (ms * 1e-3), "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": cfg.act_dtype,
                "data": "synthetic (synth/, seed 0)",
                "config": {"workload": cfg.name, "bj_config_index": cfg.bj_index, "N": cfg.N, "D": cfg.D, "L": cfg.L,
                           "H": cfg.H, "S": cfg.S, "d": cfg.d, "B": c.B, "hits": n_hit, "tau": cfg.tau,
                           "placement": args.placement, "parallelism": par, "l2": "inputs exceed L2 (no flush)",
                           **extra},
                "other_scaling": {"scaling": "strong" if args.scaling == "weak" else "weak", "B": oc.B,
                                  "ms_per_step": oms, "value": oc.B * oc.S / (oms * 1e-3), "hits": on_hit},
                "gpu_launches": launches, "clocks": clk, "warmup_steps_run": max(args.warmup, 10),
                "roofline": roof,
                "e2e": e2e}
        print(json.dumps(line), flush=True)
    del db
    ctx.close()
    dist.destroy_process_group()
    return 0


def run_e2e(args, cfg, ctx, db, step, q, Q, K, V, dev, stream):
    """The step through the public host-buffer C call (attncache_prefill_host): per step, inside the library,
    H2D of the queries, D2H of the decisions, then chunk-pipelined H2D of V (all rows) and Q/K (miss rows
    only: Alg. 2 computes q/k only on a miss), the kernels, and D2H of O.  The call is synchronous, so the
    host wall clock of K calls is the end-to-end time (CUDA events would not see the library's streams)."""
    import paper_2510_25979_b200 as ac
    qh = q.cpu().pin_memory()
    Vh = V.cpu().pin_memory()
    Qh = Q.cpu().pin_memory()
    Kh = K.cpu().pin_memory()
    Oh = torch.empty(V.shape, dtype=V.dtype).pin_memory()
    row = Vh[0].numel() * Vh.element_size()
    idx, score, hit, _ = ac.attncache_prefill_host(db, qh, Qh, Kh, Vh, cfg.tau, O=Oh)
    n_miss = int((hit == 0).sum())
    for _ in range(max(0, args.warmup - 1)):
        ac.attncache_prefill_host(db, qh, Qh, Kh, Vh, cfg.tau, O=Oh, idx=idx, score=score, hit=hit)
    torch.cuda.synchronize()
    n = max(1, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(n):
        ac.attncache_prefill_host(db, qh, Qh, Kh, Vh, cfg.tau, O=Oh, idx=idx, score=score, hit=hit)
    ms = (time.perf_counter() - t0) * 1e3 / n
    h2d = qh.numel() * qh.element_size() + Vh.numel() * Vh.element_size() + 2 * n_miss * row
    d2h = Oh.numel() * Oh.element_size() + cfg.B * (8 + 4 + 1)
    return {"value": cfg.B * cfg.S / (ms * 1e-3), "unit": "tokens/s", "ms_per_step": ms, "steps": n,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "api": "attncache_prefill_host (C ABI)",
            "copy_bound": _copy_bound(Vh, V, Qh[:n_miss], Q[:n_miss], Kh[:n_miss], K[:n_miss], Oh, ms),
            "chunk_rows": max(1, min(16, (192 << 20) // row)),
            "note": "pinned host buffers; one synchronous C-ABI call per step: chunk-pipelined copies (chunk_rows "
                    "rows, ~192 MB of V, 4-deep ring, three library streams) overlapping the kernels; one mid-call "
                    "D2H of the decisions"}


def _copy_bound(Vh, V, Qh, Q, Kh, K, Oh, e2e_ms, reps=3):
    """The PCIe floor of the e2e step, measured after it on the same buffers: the step's H2D bytes (V of every
    row, Q / K of the misses; the host copies hold the device tensors' own values) and its D2H bytes (O, the
    size of V) copied concurrently on two streams with no kernel, best of `reps`.  frac = floor / e2e step."""
    dev = V.device
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def once(h2d=True, d2h=True):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s_in):
                for d, h in ((V, Vh), (Q, Qh), (K, Kh)):
                    d.copy_(h, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s_out):
                Oh.copy_(V, non_blocking=True)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3

    both = min(once() for _ in range(reps))
    h2d_ms = min(once(d2h=False) for _ in range(reps))
    d2h_ms = min(once(h2d=False) for _ in range(reps))
    nin = sum(t.numel() * t.element_size() for t in (Vh, Qh, Kh))
    nout = Oh.numel() * Oh.element_size()
    return {"copies_only_ms": both, "frac": both / e2e_ms, "h2d_gbs_alone": nin / h2d_ms / 1e6,
            "d2h_gbs_alone": nout / d2h_ms / 1e6, "h2d_plus_d2h_gbs_concurrent": (nin + nout) / both / 1e6,
            "note": "the step's H2D and D2H bytes copied concurrently with no kernel (the e2e floor on this "
                    "host link); frac = copies_only_ms / e2e ms_per_step"}


def _ncu_traffic(cfg_name, kernel):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        t = json.load(f)
    return t.get(cfg_name, {}).get(kernel)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="llama32_1b", choices=[k for k in synth.CONFIGS if k != "search_sweep"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-search-sweep", action="store_true", help="skip the configs[4] search-QPS sweep")
    ap.add_argument("--no-target", action="store_true", help="skip the configs[2] (north_star target shape) block")
    ap.add_argument("--placement", default="affinity", choices=["affinity", "routed"],
                    help="N > 1: owner-affinity placement (default) or the literal V->owner / O->home routing")
    ap.add_argument("--scaling", default="weak", choices=["strong", "weak"],
                    help="N > 1: the config's batch on every GPU against the same sharded DB (weak, default: a serving "
                         "box answers N times the requests) or the config's global batch split over the GPUs (strong)")
    ap.add_argument("--tau", type=float, default=None, help="override the config's threshold (not for bench lines)")
    ap.add_argument("--hit-rate", type=float, default=None, help="override the config's planted hit rate")
    ap.add_argument("--batch", type=int, default=None, help="override the config's query batch")
    ap.add_argument("--seed", type=int, default=None, help="override the config's seed")
    ap.add_argument("--force-dist", action="store_true", help="run the multi-GPU path even at world size 1 (testing)")
    ap.add_argument("--aux-sms", type=int, default=0,
                    help="N > 1 pipelined step: SMs left to the side streams' search / placement / relocation kernels "
                         "(attncache_ctx_set_sm_budget; 0 = no budget, the default: at world 1 every reserve measured "
                         "slower, scripts/sm_budget_sweep.sh)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("bench.py: note: --warmup < 3 does not meet the timing rules (profiling runs only)", file=sys.stderr)
    cfg = synth.CONFIGS[args.config]
    over = {k: v for k, v in (("tau", args.tau), ("hit_rate", args.hit_rate), ("B", args.batch), ("seed", args.seed))
            if v is not None}
    if over:  # SURVEY.md §5 config overrides; the line's config then records them
        cfg = cfg.with_(**over)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: start N ranks (one process per GPU) under torch.distributed.run
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
               *(argv if argv is not None else sys.argv[1:])]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
