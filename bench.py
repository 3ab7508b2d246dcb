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
    """ncu-measured DRAM bytes per launch of the dominant kernel class (profiles/r01_traffic.json)."""
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
def cpu_reference_sample(threads: int, reps: int = 2):
    """Time the fp32 CPU oracle on a bounded sample of the config-2 workload.

    Sample: one velocity evaluation (a full denoise step) of the 2B Single-DiT
    dims at 7,800 tokens with 2 of the 28 blocks; extrapolated x14 to a full
    step and converted to cache-on steps/s with the schedule's cost model
    (a cached step runs the 7 front blocks = 0.25 of a full step).
    """
    from oracle import dit_oracle as ref
    from paper_2505_10584_b200 import SINGLE_DIT_2B, plan_cache
    from paper_2505_10584_b200.config import with_overrides
    from paper_2505_10584_b200.weights import init_weights, synthetic_inputs

    torch.set_num_threads(threads)
    cfg = with_overrides(SINGLE_DIT_2B, num_single=2)
    grid = (5, 30, 52)
    W = init_weights(cfg, seed=0)
    inp = synthetic_inputs(cfg, grid)
    orc = ref.OracleDiT(cfg, W, inp["text"], None, grid)
    x = ref.patchify(inp["x0"], cfg.patch)
    orc.velocity(x, 0.0, full=True, state={})  # warm
    ts = []
    for r in range(reps):
        t0 = time.perf_counter()
        orc.velocity(x, (r + 1) / 30, full=True, state={})
        ts.append(time.perf_counter() - t0)
    t2 = min(ts)
    t_full = t2 * (SINGLE_DIT_2B.num_layers / cfg.num_layers)
    sched = plan_cache(30)
    return {
        "full_step_s": t_full,
        "steps_per_s_cache_on": sched.speedup / t_full,
        "steps_per_s_cache_off": 1.0 / t_full,
        "sample": f"1 denoise step of Single-DiT-2B dims at 7,800 tokens with 2 of 28 blocks, best of {reps}, "
                  f"x14 extrapolated; cache-on via plan_cache(30) cost model (speedup {sched.speedup:.4f})",
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    vals = []
    t_all = time.perf_counter()
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(threads, reps=1)
        if i >= args.warmup:
            vals.append(r)
    wall = time.perf_counter() - t_all
    v = statistics.median(x["steps_per_s_cache_on"] for x in vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 30.0 / v * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "config2: Single-DiT-2B, 17x480x832 (7,800 tokens), 30 steps, cache on "
                               "(plan_cache(30)); CPU fp32 oracle port, bounded sample"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    emit(line)
    return 0


def _log(rank, msg):
    if os.environ.get("AQB_BENCH_LOG"):
        print(f"[bench r{rank} {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- our arm
def mmdit_720p(sp, timed, rank, video=None, workload=None, attention_cache=True):
    """North-star companion measurement: the 13.4B MM-DiT at BASELINE config 4's geometry
    (129x720x1280 -> 118,800 video + 256 text tokens), cache on = plan_cache(50) (24 full / 26
    cached).  One full and one cached step are timed (device events, max over ranks) after one
    warm-up of each; steps/s of the 50-step video = 50 / (24 t_full + 26 t_cached).  One more
    full step runs instrumented for the per-kernel table (joint-attention TFLOP/s).
    ``video``/``workload``: the same measurement at another geometry (config 3, 480p)."""
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
    prof = ops.KernelProfiler(timing=True)
    ops.set_profiler(prof)
    model.step("full", True)
    ops.set_profiler(None)
    kinds = prof.summary()
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
        "kernels": {k: {"ms": round(v["ms"], 2), "share": round(v["ms"] / tot, 4),
                        **({"tflops": round(v["work"] / (v["ms"] / 1e3) / 1e12, 1)}
                           if k in ("gemm", "attention") else {})}
                    for k, v in sorted(kinds.items(), key=lambda kv: -kv[1]["ms"])},
    }
    if "attention" in kinds:
        a = kinds["attention"]
        out["attention_tflops"] = a["work"] / (a["ms"] / 1e3) / 1e12
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
    del model
    torch.cuda.empty_cache()
    return out


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

    # launch count of one video, then an instrumented (per-launch CUDA events) video
    _log(rank, "profile")
    cnt = ops.KernelProfiler(timing=False)
    ops.set_profiler(cnt)
    denoise(model, x0, steps, sched_on)
    ops.set_profiler(None)
    prof = ops.KernelProfiler(timing=True)
    ops.set_profiler(prof)
    denoise(model, x0, steps, sched_on)
    ops.set_profiler(None)
    kinds = prof.summary()
    tot_ms = sum(d["ms"] for d in kinds.values())
    pk, pk_src = peaks()
    tensor_kinds = {"gemm", "attention"}
    # dominant kernel class with algorithmic work (the peer barrier moves no bytes of its own)
    dom = max((k for k in kinds if kinds[k]["work"] > 0), key=lambda k: kinds[k]["ms"])
    d = kinds[dom]
    if dom in tensor_kinds:
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
        if k in tensor_kinds:
            e["tflops"] = round(v["work"] / (v["ms"] / 1e3) / 1e12, 1)
        elif v["work"] > 0:
            e["gbs"] = round(v["work"] / (v["ms"] / 1e3) / 1e9, 1)
        per_kind[k] = e
    attn = kinds.get("attention")
    attn_tflops = attn["work"] / (attn["ms"] / 1e3) / 1e12 if attn else None

    fl = flops_per_step(cfg, grid[0] * grid[1] * grid[2])
    mm = mm480 = None
    if not args.no_mmdit:
        _log(rank, "mmdit 720p")
        del model, graphs
        torch.cuda.empty_cache()
        from paper_2505_10584_b200.config import VIDEO_480P_61F
        mm_sp = sp  # TP-SP (--parallel tp) covers both families
        mm = mmdit_720p(mm_sp, timed, rank)
        mm480 = mmdit_720p(mm_sp, timed, rank, VIDEO_480P_61F,
                           "config3: MM-DiT-13.4B, 61x480x848 -> 25,440 video + 256 text tokens, 50 Euler steps, "
                           "cache on = plan_cache(50) (24 full / 26 cached)", attention_cache=False)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_on / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "config2: Single-DiT-2B (fitted H=2048 A=16 L=28), 17x480x832 -> 7,800 tokens, "
                                   "text 256x4096, 30 Euler steps, cache on = plan_cache(30) (17 full/13 cached); "
                                   "1 bench step = 1 video",
                       "parallelism": (f"tp{world}-sp" if args.parallel == "tp" else f"ulysses-sp{world}")
                       if world > 1 else "single-gpu",
                       "tp_exchange": ("p2p: all-gather stored by the LN+modulate kernel into every rank, "
                                       "reduce-scatter as TMA reduce-add from the row-parallel GEMM epilogues; "
                                       "device barrier") if (sp and sp.tensor_parallel) else None,
                       "ulysses_exchange": None if (sp and sp.tensor_parallel) else (sp.exchange + (" (QKV-GEMM and attention epilogues store into peer "
                                            "memory over NVLink; device barrier)" if sp.exchange == "p2p" else
                                            " all_to_all")) if sp else None,
                       "l2": "inputs larger than L2 (4.3 GB of bf16 weights streamed per step)",
                       "cuda_graphs": bool(args.graph),
                       "pdl": os.environ.get("AQB_PDL", "1") != "0"},
            "cache_off": {"value": value_off, "unit": UNIT, "ms_per_video": ms_off / max(1, args.steps)},
            "cache_speedup_measured": value / value_off,
            "schedule": sched_on.as_string(),
            "attention_tflops": attn_tflops,
            "model_tflops_full_step": fl["total"] / (ms_off / max(1, args.steps) / steps / 1e3) / 1e12,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": out_bytes, "d2h_bytes_per_step": out_bytes},
            "gpu_launches": cnt.count * args.steps,
            "roofline": roof,
            "kernels": per_kind,
            "clocks": clocks,
        }
        if mm is not None:
            line["mmdit_720p"] = mm
            line["mmdit_480p"] = mm480
        if world == 1 and not args.no_cpu:
            threads = os.cpu_count() or 1
            c = cpu_reference_sample(threads)
            line["cpu_baseline"] = {"value": c["steps_per_s_cache_on"], "unit": UNIT, "cores": threads, "kind": "port",
                                    "sample": c["sample"]}
        emit(line)
    _log(rank, "done")
    if sp:
        dist.barrier()
        torch.cuda.synchronize()
    sys.stdout.flush()
    sys.stderr.flush()
    # NCCL communicators captured inside CUDA graphs can make process-group
    # teardown block; the job's results are already printed, so exit hard.
    os._exit(0)


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
