#!/usr/bin/env python
"""Benchmark: DiT denoise steps/sec on B200 (BASELINE.json metric).

Workload (N=1 and every N): BASELINE config 2 — Single-DiT 2B (fitted dims
H=2048, 16 heads, 28 blocks, mT5-XXL-sized text 256x4096), one 17x480x832
video (latent 8x5x60x104 -> 7,800 tokens), 30 Euler steps, diffusion cache ON
(``plan_cache(30)``: 17 full / 13 cached).  One bench "step" = one complete
30-step denoise of one video; ``value`` = denoise steps/s of the whole job.
N > 1 runs the same video with Ulysses sequence parallelism (strong scaling).

Also reported: cache-OFF steps/s, ``e2e`` through the public API with the
noise latent in pinned host memory (H2D + final D2H inside the timed region),
the dominant kernel's roofline (CUDA events around every launch in an
instrumented pass), launch count, SM clocks sampled during the timed region,
and the CPU reference path (the fp32 oracle, ``oracle/``) timed on this
host's cores on a bounded sample.

``--impl reference`` times that CPU reference path alone (rank 0).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DiT denoise steps/sec & attention TFLOPS at 1/2/4/8 B200 vs CPU ref"
UNIT = "denoise_steps/s"
PEAK_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def traffic(kind):
    """ncu-measured DRAM bytes per launch of the dominant kernel class (profiles/r02_traffic.json,
    the final round-2 captures; r01_traffic.json if absent)."""
    p = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if not os.path.exists(p):
        p = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as fh:
        d = json.load(fh).get(kind)
    return (d["dram_bytes_per_launch"], d) if d else (None, None)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d, "measured"
    return PEAK_FALLBACK, "fallback"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------- CPU reference path
# The reference has no executable DiT; its CPU path for this metric is the fp32
# restatement in oracle/ (test infrastructure, executed only here, in the cpu_baseline leg and in
# --impl reference).  BASELINE.md's plan: config 2 measured on full-depth steps, configs 3-4 from
# per-block timings fitted a*S^2 + b*S (labelled extrapolated), config 5 as fp32 SDPA.

CONFIG2_GRID = (5, 30, 52)
CONFIG2_STEPS = 30


def _oracle_config2():
    from oracle import dit_oracle as ref
    from paper_2505_10584_b200 import SINGLE_DIT_2B, front_block_count
    from paper_2505_10584_b200.weights import init_weights, synthetic_inputs

    cfg = SINGLE_DIT_2B
    W = init_weights(cfg, seed=0)
    inp = synthetic_inputs(cfg, CONFIG2_GRID)
    orc = ref.OracleDiT(cfg, W, inp["text"], None, CONFIG2_GRID, n_front=front_block_count(cfg.num_layers, 0.25))
    del W
    return cfg, orc, ref.patchify(inp["x0"], cfg.patch)


def cpu_config2_measured(threads: int, full_steps: int = 2) -> dict:
    """Config 2 on the CPU oracle, measured end to end: ``full_steps`` full 28-block denoise
    steps (velocity + Euler, real data flow) then one cached step (front 7 blocks + the rear
    offset), fp32 on ``threads`` cores.  Cache-on steps/s of the 30-step video =
    30 / (17·t_full + 13·t_cached) with plan_cache(30)'s flags."""
    from paper_2505_10584_b200 import plan_cache

    torch.set_num_threads(threads)
    cfg, orc, x = _oracle_config2()
    sched = plan_cache(CONFIG2_STEPS)
    state, t_full = {}, []
    with torch.no_grad():
        for s in range(full_steps):
            t0 = time.perf_counter()
            v, _ = orc.velocity(x, s / CONFIG2_STEPS, full=True, state=state)
            x = x + v / CONFIG2_STEPS
            t_full.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        v, _ = orc.velocity(x, full_steps / CONFIG2_STEPS, full=False, state=state)
        t_cached = time.perf_counter() - t0
    tf = statistics.mean(t_full)
    video_s = sched.full_steps * tf + sched.cached_steps * t_cached
    return {
        "steps_per_s_cache_on": CONFIG2_STEPS / video_s, "steps_per_s_cache_off": 1.0 / tf,
        "full_step_s": t_full, "cached_step_s": t_cached,
        "sample": f"config 2 measured: {full_steps} full 28-block denoise steps + 1 cached step (7 front blocks) "
                  f"of the fp32 oracle at 7,800 tokens; cache on = 30 / (17 t_full + 13 t_cached)",
    }


def cpu_mmdit_fit(threads: int, sizes=(8192, 16384)) -> dict:
    """Configs 3-4 (MM-DiT 13.4B, 25 dual + 29 single blocks): one dual-stream and one joint
    block timed on the CPU oracle at ``sizes`` video tokens (+256 text), each fitted
    t(S) = a·S² + b·S, then extrapolated to the full sequence × 54 blocks.  EXTRAPOLATED."""
    from oracle import dit_oracle as ref
    from paper_2505_10584_b200 import MM_DIT_13B, front_block_count, plan_cache
    from paper_2505_10584_b200.config import VIDEO_480P_61F, VIDEO_720P_129F, with_overrides
    from paper_2505_10584_b200.weights import init_weights

    torch.set_num_threads(threads)
    cfg = with_overrides(MM_DIT_13B, num_dual=1, num_single=1)
    W = {k: v.float() for k, v in init_weights(cfg, seed=0).items()}
    H, St = cfg.hidden_size, cfg.text_len
    g = torch.Generator().manual_seed(1)
    vec = torch.randn(H, generator=g)
    meas = {"dual": [], "single": []}
    with torch.no_grad():
        warm = torch.randn(1024, H, generator=g)  # first-call allocation / thread-pool warm-up
        ref.mm_dual_block(W, 0, warm, warm[:St], vec, cfg, ref.rope_angles((1, 32, 32), cfg.rope_dims, cfg.rope_theta))
        for Sv in sizes:
            grid = (Sv // 1024, 32, 32)
            ang = ref.rope_angles(grid, cfg.rope_dims, cfg.rope_theta)
            img = torch.randn(Sv, H, generator=g)
            txt = torch.randn(St, H, generator=g)
            t0 = time.perf_counter()
            img2, txt2, _ = ref.mm_dual_block(W, 0, img, txt, vec, cfg, ang)
            meas["dual"].append(time.perf_counter() - t0)
            x = torch.cat([img2, txt2])
            t0 = time.perf_counter()
            ref.mm_single_block(W, 0, x, vec, cfg, ang)
            meas["single"].append(time.perf_counter() - t0)
    S = [sv + St for sv in sizes]
    fit = {}
    for kind, ts in meas.items():
        # t = a S^2 + b S through the two measured points
        (s1, s2), (t1, t2) = S, ts
        a = (t2 / s2 - t1 / s1) / (s2 - s1)
        fit[kind] = (a, t1 / s1 - a * s1)
    L = MM_DIT_13B
    nf = front_block_count(L.num_layers, 0.25)
    sched = plan_cache(50)
    out = {"measured_block_s": {k: dict(zip([str(s) for s in S], v)) for k, v in meas.items()},
           "fit_a_b": {k: list(v) for k, v in fit.items()}}
    for name, video in (("config3_480p", VIDEO_480P_61F), ("config4_720p", VIDEO_720P_129F)):
        Sfull = video.tokens(L) + St
        td = fit["dual"][0] * Sfull ** 2 + fit["dual"][1] * Sfull
        ts_ = fit["single"][0] * Sfull ** 2 + fit["single"][1] * Sfull
        t_full = L.num_dual * td + L.num_single * ts_
        t_cached = min(nf, L.num_dual) * td + max(0, nf - L.num_dual) * ts_
        video_s = sched.full_steps * t_full + sched.cached_steps * t_cached
        out[name] = {"tokens": Sfull, "full_step_s_extrapolated": t_full, "cached_step_s_extrapolated": t_cached,
                     "steps_per_s_cache_on_extrapolated": 50 / video_s}
    out["sample"] = (f"EXTRAPOLATED: one dual + one joint MM-DiT-13.4B block (H=3072, 24 heads) timed on the fp32 "
                     f"oracle at {'/'.join(str(s) for s in sizes)} video + 256 text tokens, t(S) = a S^2 + b S per "
                     f"block kind, x (25 dual + 29 single) at the full sequence; plan_cache(50) 24 full / 26 cached "
                     f"(14 front blocks)")
    return out


def cpu_sdpa(threads: int, sizes=(4096, 8192), heads: int = 24, head_dim: int = 128) -> dict:
    """Config 5 on the CPU: fp32 softmax(QKᵀ/√d)V (the oracle's attention), B=1, 24 heads × 128,
    non-causal; TFLOP/s by the 4·S²·d·heads convention."""
    from oracle import dit_oracle as ref

    torch.set_num_threads(threads)
    g = torch.Generator().manual_seed(0)
    out = {}
    with torch.no_grad():
        for S in sizes:
            q, k, v = (torch.randn(S, heads, head_dim, generator=g) for _ in range(3))
            t0 = time.perf_counter()
            ref.attention(q, k, v)
            dt = time.perf_counter() - t0
            out[str(S)] = {"s": dt, "tflops": 4.0 * S * S * head_dim * heads / dt / 1e12}
    return out


def cpu_baseline_full(threads: int) -> dict:
    c2 = cpu_config2_measured(threads)
    mm = cpu_mmdit_fit(threads)
    sd = cpu_sdpa(threads)
    return {"value": c2["steps_per_s_cache_on"], "unit": UNIT, "cores": threads, "kind": "port",
            "sample": c2["sample"], "config2": c2, "mmdit_extrapolated": mm, "config5_sdpa_fp32": sd}


def run_reference(args):
    """The reference CPU path for the same metric/config as our arm: config 2's denoise steps/s
    (cache on), composed from measured per-block samples.  Each bench step runs the embed, two
    of the 28 blocks (rotating through all of them, each on its own weights, full size) and the
    final layer of one full denoise step; a full step = embed/final + the 28 blocks' measured
    times, a cached step = embed/final + the 7 front blocks, the video = 17 full + 13 cached."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2505_10584_b200 import front_block_count, plan_cache

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    t_all = time.perf_counter()
    cfg, orc, x = _oracle_config2()
    L = cfg.num_layers
    per_block = {i: [] for i in range(L)}
    shell, samples = [], []
    with torch.no_grad():
        t0 = time.perf_counter()
        orc.run_blocks(x, 0.0, [])  # embed + final alone
        shell.append(time.perf_counter() - t0)
        for it in range(args.warmup + args.steps):
            ids = [(2 * it) % L, (2 * it + 1) % L]
            t0 = time.perf_counter()
            orc.run_blocks(x, 0.5, ids)
            dt = time.perf_counter() - t0
            if it >= args.warmup:
                samples.append(dt)
            for i in ids:  # the block's share: sample minus the embed/final shell, split evenly
                per_block[i].append((dt - shell[0]) / 2)
    missing = [i for i in range(L) if not per_block[i]]
    blk = {i: statistics.median(v) for i, v in per_block.items() if v}
    mean_blk = statistics.mean(blk.values())
    for i in missing:  # fewer than 14 samples in total: unseen blocks take the mean (same shape)
        blk[i] = mean_blk
    t_full = shell[0] + sum(blk.values())
    t_cached = shell[0] + sum(blk[i] for i in range(front_block_count(L, 0.25)))
    sched = plan_cache(CONFIG2_STEPS)
    v = CONFIG2_STEPS / (sched.full_steps * t_full + sched.cached_steps * t_cached)
    wall = time.perf_counter() - t_all
    sample = (f"per bench step: embed + 2 of the 28 Single-DiT-2B blocks (rotating over all blocks, full "
              f"7,800-token size, own weights) + final of the fp32 oracle; video composed from the measured "
              f"blocks as 17 full (28 blocks) + 13 cached (7 front blocks) steps; {L - len(missing)}/28 blocks measured")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.mean(samples) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(),
        "reference_path": "fp32 CPU restatement of the DiT (oracle/dit_oracle.py): the reference ditplan has no "
                          "executable DiT, only the cache schedule (bit-exact in the product)",
        "ms_full_step_composed": t_full * 1e3, "ms_cached_step_composed": t_cached * 1e3,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    emit(line)
    return 0


def config_dict():
    """The workload both arms measure (identical dict in both JSON lines)."""
    return {"workload": "config2: Single-DiT-2B (fitted H=2048 A=16 L=28), 17x480x832 -> 7,800 tokens, "
                        "text 256x4096, 30 Euler steps, cache on = plan_cache(30) (17 full/13 cached); "
                        "1 bench step = 1 video",
            "global_batch": 1, "seq_len": 7800,
            "l2": "inputs larger than L2 (4.3 GB of bf16 weights streamed per denoise step)"}


def _log(rank, msg):
    if os.environ.get("AQB_BENCH_LOG"):
        print(f"[bench r{rank} {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- our arm
def mmdit_720p(sp, timed, rank, video=None, workload=None, attention_cache=True, full_video=False):
    """North-star companion measurement: the 13.4B MM-DiT at BASELINE config 4's geometry
    (129x720x1280 -> 118,800 video + 256 text tokens), cache on = plan_cache(50) (24 full / 26
    cached).  One full and one cached step are timed (device events, max over ranks) after one
    warm-up of each; steps/s of the 50-step video = 50 / (24 t_full + 26 t_cached).  One more
    full step runs instrumented for the per-kernel table (joint-attention TFLOP/s).
    ``video``/``workload``: the same measurement at another geometry (config 3, 480p).
    ``full_video``: also time one complete 50-step denoise (CUDA graphs) through the public
    ``denoise`` API — measured, not composed (config 3 by default; 720p with --mmdit-full-video)."""
    from paper_2505_10584_b200 import MM_DIT_13B, build_model, flops_per_step, ops, plan_cache
    from paper_2505_10584_b200.config import VIDEO_720P_129F
    from paper_2505_10584_b200.weights import init_weights, synthetic_inputs

    cfg = MM_DIT_13B
    grid = (video or VIDEO_720P_129F).grid(cfg)
    steps = 50
    sched = plan_cache(steps)
    W = init_weights(cfg, seed=0, device="cuda")
    inp = synthetic_inputs(cfg, grid, device="cuda")
    model = build_model(cfg, weights=W, sp=sp).prepare(grid, inp["text"], inp["pooled"])
    del W
    torch.cuda.empty_cache()
    model.reset(inp["x0"], steps)
    model.step("full", True)
    model.step("cached", True)
    t_full = timed(lambda: model.step("full", True), 1)
    t_cached = timed(lambda: model.step("cached", True), 1)
    kinds, method, _ = kernel_table(lambda: model.step("full", True))
    tot = sum(d["ms"] for d in kinds.values())
    n_full, n_cached = sched.full_steps, sched.cached_steps
    video_ms = n_full * t_full + n_cached * t_cached
    fl = flops_per_step(cfg, grid[0] * grid[1] * grid[2])
    out = {
        "workload": workload or ("config4: MM-DiT-13.4B (fitted H=3072 A=24, 25 dual + 29 single), 129x720x1280 -> "
                                 "118,800 video + 256 text tokens, 50 Euler steps, cache on = plan_cache(50) "
                                 "(24 full / 26 cached)"),
        "value": steps / (video_ms / 1e3), "unit": "denoise_steps/s",
        "ms_full_step": t_full, "ms_cached_step": t_cached,
        "model_tflops_full_step": fl["total"] / (t_full / 1e3) / 1e12,
        "kernel_timing": method,
        "kernels": {k: {"ms": round(v["ms"], 2), "share": round(v["ms"] / tot, 4),
                        **({"tflops": round(v["work"] / (v["ms"] / 1e3) / 1e12, 1)}
                           if k in ("gemm", "attention") else {})}
                    for k, v in sorted(kinds.items(), key=lambda kv: -kv[1]["ms"])},
    }
    if "attention" in kinds:
        a = kinds["attention"]
        out["attention_tflops"] = a["work"] / (a["ms"] / 1e3) / 1e12
    if full_video:
        from paper_2505_10584_b200 import denoise
        from paper_2505_10584_b200.sampler import _Graphs

        gr = _Graphs()
        run = lambda: denoise(model, inp["x0"], steps, sched, graph=True, graphs=gr)  # noqa: E731
        run()  # captures the full- and the cached-step graph
        t_video = timed(run, 1)
        gr.clear()
        out["measured_video"] = {"value": steps / (t_video / 1e3), "unit": "denoise_steps/s", "ms_per_video": t_video,
                                 "note": "one complete plan_cache(50) denoise through denoise(..., graph=True)"}
    if attention_cache and not getattr(sp, "tensor_parallel", False):
        # the paper's second cache mode: every block runs, cached steps reuse each
        # block's attention output (the 86% FLOP share at 720p) — same plan_cache(50) schedule
        sched_ac = plan_cache(steps, mode="attention-cache")
        model.reset(inp["x0"], steps, cache_mode="attention-cache")
        model.step("full", True)
        model.step("cached", True)
        ta_full = timed(lambda: model.step("full", True), 1)
        ta_cached = timed(lambda: model.step("cached", True), 1)
        ac_ms = sched_ac.full_steps * ta_full + sched_ac.cached_steps * ta_cached
        out["attention_cache"] = {"value": steps / (ac_ms / 1e3), "unit": "denoise_steps/s",
                                  "ms_full_step": ta_full, "ms_cached_step": ta_cached,
                                  "speedup_vs_no_cache": steps * t_full / ac_ms}
        out["dit_layer_cache_speedup_vs_no_cache"] = steps * t_full / video_ms
    out["peer_barriers_ok"] = model.peer_ok()
    model.close()
    del model
    torch.cuda.empty_cache()
    return out


TENSOR_KINDS = ("gemm", "attention")


def kernel_table(run):
    """Per kind: launches, device ms and algorithmic work (FLOPs / HBM bytes) of one ``run()``.

    Work comes from the launch records (``ops.KernelProfiler``); time from a CUPTI trace of a
    second run (``ops.trace_kernels``: each kernel's own execution, PDL off).  If the tracer is
    unavailable, CUDA events around every launch are used instead (they include launch gaps).
    Returns (kinds, method, libaqb kernels launched)."""
    from paper_2505_10584_b200 import ops

    cnt = ops.KernelProfiler(timing=False)
    ops.set_profiler(cnt)
    run()
    ops.set_profiler(None)
    kinds = {k: dict(v) for k, v in cnt.summary().items()}
    try:
        tr = ops.trace_kernels(run)
        if not tr:
            raise RuntimeError("empty trace")
        for k, v in tr.items():
            d = kinds.setdefault(k, {"launches": 0, "ms": 0.0, "work": 0.0})
            d["launches"], d["ms"] = v["launches"], v["ms"]
        method = "CUPTI kernel durations (torch.profiler), PDL off, eager launches"
        n = sum(v["launches"] for v in tr.values())
    except Exception as e:  # pragma: no cover - tracer missing on the box
        ev = ops.KernelProfiler(timing=True)
        ops.set_profiler(ev)
        run()
        ops.set_profiler(None)
        kinds = ev.summary()
        method = f"CUDA events around every launch (tracer unavailable: {e})"
        n = cnt.count
    kinds = {k: v for k, v in kinds.items() if v["ms"] > 0}
    return kinds, method, n


def roofline(kinds):
    """Roofline of the dominant kernel class with algorithmic work, and the per-kind table."""
    tot_ms = sum(d["ms"] for d in kinds.values())
    pk, pk_src = peaks()
    dom = max((k for k in kinds if kinds[k]["work"] > 0), key=lambda k: kinds[k]["ms"])
    d = kinds[dom]
    if dom in TENSOR_KINDS:
        ach = d["work"] / (d["ms"] / 1e3) / 1e12
        peak = pk["bf16_tflops_sustained"]
        tb, tinfo = traffic(dom)
        roof = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "traffic": tb, "peak_source": f"{pk_src} bf16 sustained",
                "share_of_step": d["ms"] / tot_ms}
        if tinfo:
            roof["traffic_note"] = (f"{tinfo['kernel']}: {tb / 1e6:.1f} MB DRAM per launch vs "
                                    f"{tinfo['algorithmic_bytes_per_launch'] / 1e6:.1f} MB algorithmic ({tinfo['source']})")
    else:
        ach = d["work"] / (d["ms"] / 1e3) / 1e9
        peak = pk["hbm_gbs"]
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": None, "peak_source": f"{pk_src} hbm copy", "share_of_step": d["ms"] / tot_ms}
    per_kind = {}
    for k, v in sorted(kinds.items(), key=lambda kv: -kv[1]["ms"]):
        e = {"launches": v["launches"], "ms": round(v["ms"], 3), "share": round(v["ms"] / tot_ms, 4)}
        if k in TENSOR_KINDS and v["work"] > 0:
            e["tflops"] = round(v["work"] / (v["ms"] / 1e3) / 1e12, 1)
        elif v["work"] > 0:
            e["gbs"] = round(v["work"] / (v["ms"] / 1e3) / 1e9, 1)
        per_kind[k] = e
    return roof, per_kind


def run_ours(args):
    from paper_2505_10584_b200 import SINGLE_DIT_2B, build_model, denoise, no_cache, plan_cache, flops_per_step
    from paper_2505_10584_b200 import ops
    from paper_2505_10584_b200.parallel import TensorSP, Ulysses, init_from_env, local_device_index
    from paper_2505_10584_b200.sampler import _Graphs
    from paper_2505_10584_b200.weights import init_weights, synthetic_inputs
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = local_device_index()
    sp = None
    if world > 1:
        init_from_env("nccl")
        sp = TensorSP() if args.parallel == "tp" else Ulysses()
    torch.cuda.set_device(local)
    rank = sp.rank if sp else 0
    cfg = SINGLE_DIT_2B
    grid = (5, 30, 52)
    steps = 30
    sched_on = plan_cache(steps)
    sched_off = no_cache(steps)
    W = init_weights(cfg, seed=0, device="cuda")
    inp = synthetic_inputs(cfg, grid, device="cuda")
    model = build_model(cfg, weights=W, sp=sp).prepare(grid, inp["text"])
    del W
    x0 = inp["x0"]
    graphs = _Graphs()

    def barrier():
        if sp:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, k):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        if sp:
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        barrier()
        return float(ms)

    run_on = lambda: denoise(model, x0, steps, sched_on, graph=args.graph, graphs=graphs)  # noqa: E731
    run_off = lambda: denoise(model, x0, steps, sched_off, graph=args.graph, graphs=graphs)  # noqa: E731
    _log(rank, "warmup")
    for _ in range(args.warmup):
        run_on()
    run_off()
    torch.cuda.synchronize()

    _log(rank, "timed")
    clk = ClockSampler(local)
    clk.start()
    ms_on = timed(run_on, args.steps)
    clocks = clk.stop()
    ms_off = timed(run_off, max(1, args.steps))
    value = steps * args.steps / (ms_on / 1e3)
    value_off = steps * max(1, args.steps) / (ms_off / 1e3)

    # e2e through the public API: pinned host latent in, host latent out
    _log(rank, "e2e")
    x0_host = x0.cpu().pin_memory()
    out_bytes = x0_host.numel() * 4

    def e2e_once():
        res = denoise(model, x0_host, steps, sched_on, graph=args.graph, graphs=graphs)
        res.latent.cpu()

    e2e_once()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_once()
    barrier()
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], device="cuda")
    if sp:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = steps * args.steps / float(e2e_t)

    # per-kernel table of one video: algorithmic work per kind from the launch records,
    # device time per kind from a CUPTI trace of the same video (PDL off)
    _log(rank, "profile")
    kinds, timing_method, n_kernels = kernel_table(lambda: denoise(model, x0, steps, sched_on))
    roof, per_kind = roofline(kinds)
    attn = kinds.get("attention")
    attn_tflops = attn["work"] / (attn["ms"] / 1e3) / 1e12 if attn else None

    fl = flops_per_step(cfg, grid[0] * grid[1] * grid[2])
    peer_ok = model.peer_ok()
    mm = mm480 = None
    if not args.no_mmdit:
        _log(rank, "mmdit 720p")
        graphs.clear()
        graphs = None
        model.close()
        model = None
        torch.cuda.empty_cache()
        from paper_2505_10584_b200.config import VIDEO_480P_61F
        mm_sp = sp  # TP-SP (--parallel tp) covers both families
        mm = mmdit_720p(mm_sp, timed, rank, full_video=args.mmdit_full_video)
        mm480 = mmdit_720p(mm_sp, timed, rank, VIDEO_480P_61F,
                           "config3: MM-DiT-13.4B, 61x480x848 -> 25,440 video + 256 text tokens, 50 Euler steps, "
                           "cache on = plan_cache(50) (24 full / 26 cached)", attention_cache=False, full_video=True)
    if mm is not None:
        peer_ok = peer_ok and mm["peer_barriers_ok"] and mm480["peer_barriers_ok"]
    # every rank: a peer barrier that timed out means a rank never arrived — the numbers are void
    ok = torch.tensor([1 if peer_ok else 0], device="cpu" if sp and dist.get_backend() == "gloo" else "cuda")
    if sp:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if int(ok) != 1:
        raise RuntimeError("peer barrier timed out during the bench (a rank never arrived); no result")
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_on / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": config_dict(),
            "parallelism": (f"tp{world}-sp" if args.parallel == "tp" else f"ulysses-sp{world}")
            if world > 1 else "single-gpu",
            "exchange": exchange_note(sp),
            "launch": {"cuda_graphs": bool(args.graph), "pdl": os.environ.get("AQB_PDL", "1") != "0"},
            "cache_off": {"value": value_off, "unit": UNIT, "ms_per_video": ms_off / max(1, args.steps)},
            "cache_speedup_measured": value / value_off,
            "schedule": sched_on.as_string(),
            "attention_tflops": attn_tflops,
            "model_tflops_full_step": fl["total"] / (ms_off / max(1, args.steps) / steps / 1e3) / 1e12,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": out_bytes, "d2h_bytes_per_step": out_bytes},
            "gpu_launches": n_kernels * args.steps,
            "kernel_timing": timing_method,
            "roofline": roof,
            "kernels": per_kind,
            "clocks": clocks,
            "peer_barriers_ok": True,
        }
        if mm is not None:
            line["mmdit_720p"] = mm
            line["mmdit_480p"] = mm480
        if world == 1 and not args.no_cpu:
            _log(rank, "cpu baseline")
            line["cpu_baseline"] = cpu_baseline_full(os.cpu_count() or 1)
        emit(line)
    _log(rank, "teardown")
    # orderly teardown (the driver reads which libraries this process mapped at exit): graphs
    # first (they hold peer-buffer addresses), then the collective peer-buffer release, then
    # the process group.  The default p2p exchange captures no NCCL call in a graph.
    graphs = None
    if model is not None:
        model.close()
        model = None
    if sp:
        dist.barrier()
        torch.cuda.synchronize()
        dist.destroy_process_group()
    torch.cuda.synchronize()
    sys.stdout.flush()
    sys.stderr.flush()
    return 0


def exchange_note(sp):
    if sp is None:
        return None
    if sp.tensor_parallel:
        return ("TP-SP p2p: all-gather stored by the LN+modulate kernel into every rank, reduce-scatter as TMA "
                "reduce-add from the row-parallel GEMM epilogues; device barrier")
    if sp.exchange == "p2p":
        return "Ulysses p2p: QKV-GEMM and attention epilogues store into peer memory over NVLink; device barrier"
    return "Ulysses NCCL all_to_all"


_JSON_OUT = None


def emit(line: dict):
    """The one JSON line on the real stdout (library chatter, e.g. NCCL's version banner, goes to stderr)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)  # fd 1 (C and Python prints) -> stderr for the rest of the run
    sys.stdout = sys.stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-mmdit", action="store_true", help="skip the 13.4B MM-DiT 720p companion measurement")
    ap.add_argument("--mmdit-full-video", action="store_true",
                    help="also time a complete 50-step 720p MM-DiT video (about 4.5 min at N=1)")
    ap.add_argument("--parallel", choices=["ulysses", "tp"], default="ulysses",
                    help="N>1: Ulysses sequence parallel (default) or TP-SP (both families)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
