#!/usr/bin/env python
"""Benchmark of the tiled MonarchAttention forward (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--config sf] [--impl ours|reference]

A step is one tiled MonarchAttention forward over one synthetic layer of the
configured workload (default C2: one Self-Forcing chunk, B=1 H=12 d=128,
(f,h,w)=(3,30,52), (h,w)-tiled plan, T=1, bf16).  Multi-GPU runs partition the
flattened (b,h) unit list with ``shard.head_shard`` (no
collective in the data path):

* C2-C4 (``sf``, ``kv21``, ``n32k`` ...): weak scaling -- the job holds N
  layers' worth of units (global batch N), each rank owns the contiguous span
  of B*H units of one layer; ``value`` = whole-job ms per layer = max-over-ranks
  device time per step / N.
* C5 (``wan``): strong scaling of one fixed workload -- the Wan-1.3B-shaped
  30-layer attention stack, B=8 H=12 N=32760, 96 (b,h) units split over the
  ranks; ``value`` = ms per 30-layer stack (max over ranks).  The optional
  NCCL all-gather of each layer's output shards (sequence-parallel DiT block)
  is timed separately.

``python bench.py --gpus N`` without a torchrun environment re-launches itself
under ``torch.distributed.run`` with N ranks (127.0.0.1 rendezvous).

Timing: W warm-up steps, then K steps timed with CUDA events on the launching
stream; a 256 MB buffer is rewritten between steps to flush L2 (126 MB), and
the flush is outside the timed events.  Dense attention on the same shape
(cuDNN SDPA, flash_attn, flashinfer) is timed identically; the fastest is the
"dense FA" denominator.  ``--impl reference`` times the unmodified reference
CPU implementation (baseline/_ref, falling back to the oracle port) on the
host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MonarchAttn fwd ms/layer at Self-Forcing shape; speedup vs dense FA; TC util %"

CONFIGS = {
    # name: (B, H, f_kv, f_q, h, w, d, neighborhoods, dtype, description)
    "sf": (1, 12, 3, 3, 30, 52, 128, (1, 30, 52), "bf16",
           "C2 Self-Forcing chunk: B=1 H=12 d=128, 3 frames x 1560 tokens, (h,w)-tiled plan"),
    "sf3hw": (1, 12, 3, 3, 30, 52, 128, (3, 30, 52), "bf16",
              "C2' Self-Forcing chunk, (3h,w) plan = untiled (90,52)"),
    "kv21": (1, 12, 21, 3, 30, 52, 128, (1, 30, 52), "bf16",
             "C3 chunked-KV rollout: 3 query frames vs 21 KV frames, (h,w)-tiled"),
    "n32k": (1, 12, 21, 21, 30, 52, 128, (1, 30, 52), "bf16",
             "C4 N=32760 (21,30,52), (h,w)-tiled G=21"),
    "kv21_3hw": (1, 12, 21, 3, 30, 52, 128, (3, 30, 52), "bf16",
                 "C3b chunked-KV rollout: 3 query frames vs 21 KV frames, (3h,w)-tiled (paper's s=0.97)"),
    "n32k_3hw": (1, 12, 21, 21, 30, 52, 128, (3, 30, 52), "bf16",
                 "C4b N=32760 (21,30,52), (3h,w)-tiled G=7 (paper's Wan 480p s=0.97)"),
    "n32k_fhw": (1, 12, 21, 21, 30, 52, 128, None, "bf16",
                 "C4c N=32760 untiled aligned (fh,w) = (630,52)"),
    "n32k_mis": (1, 12, 21, 21, 30, 52, 128, "mis", "bf16",
                 "C4d N=32760 untiled misaligned raw (b1,b2) = (1260,26)"),
    "n32k_f": (1, 12, 21, 21, 30, 52, 128, ("aligned", ("f",)), "bf16",
               "C4e N=32760 untiled aligned (f, hw) = (21,1560) (long tile rows: online-softmax row stage)"),
    "n32k_w": (1, 12, 21, 21, 30, 52, 128, ("aligned", ("w",)), "bf16",
               "C4f N=32760 untiled aligned (w, fh) = (52,630) (permuted plan: gathered into slot order)"),
    "n32k_hw": (1, 12, 21, 21, 30, 52, 128, ("aligned", ("h", "w")), "bf16",
                "C4g N=32760 untiled aligned (hw, f) = (1560,21) (permuted plan: gathered into slot order)"),
    "n32k_fw": (1, 12, 21, 21, 30, 52, 128, ("aligned", ("f", "w")), "bf16",
                "C4h N=32760 untiled aligned (fw, h) = (1092,30) (permuted plan: gathered into slot order)"),
    "n32k_h": (1, 12, 21, 21, 30, 52, 128, ("aligned", ("h",)), "bf16",
               "C4i N=32760 untiled aligned (h, fw) = (30,1092) (permuted plan: gathered into slot order)"),
    "sf720": (1, 12, 3, 3, 45, 80, 128, (1, 45, 80), "bf16",
              "720p Self-Forcing chunk: B=1 H=12, 3 frames x (45,80), (h,w)-tiled (PAPER.md:866 shapes)"),
    "sf720_3hw": (1, 12, 3, 3, 45, 80, 128, (3, 45, 80), "bf16",
                  "720p Self-Forcing chunk, (3h,w) plan"),
    "kv21_720": (1, 12, 21, 3, 45, 80, 128, (1, 45, 80), "bf16",
                 "720p chunked-KV rollout: 3 query frames vs 21 KV frames of (45,80), (h,w)-tiled (paper s=0.97)"),
    "kv21_720_3hw": (1, 12, 21, 3, 45, 80, 128, (3, 45, 80), "bf16",
                     "720p chunked-KV rollout, (3h,w)-tiled (paper s=0.98)"),
    "n75k_720": (1, 12, 21, 21, 45, 80, 128, (1, 45, 80), "bf16",
                 "Wan 720p layer: N=75600 (21,45,80), (h,w)-tiled (PAPER.md:837, s=0.97)"),
    "n75k_720_3hw": (1, 12, 21, 21, 45, 80, 128, (3, 45, 80), "bf16",
                     "Wan 720p layer: N=75600 (21,45,80), (3h,w)-tiled (PAPER.md:837, s=0.98)"),
    "wan": (8, 12, 21, 21, 30, 52, 128, (1, 30, 52), "bf16",
            "C5 Wan-1.3B-shaped attention stack: 30 layers x B=8 H=12 N=32760 (h,w)-tiled (s=0.95), "
            "96 (b,h) units head-sharded over the ranks"),
    "wan_3hw": (8, 12, 21, 21, 30, 52, 128, (3, 30, 52), "bf16",
                "C5b Wan-1.3B-shaped attention stack: 30 layers x B=8 H=12 N=32760 (3h,w)-tiled (s=0.97), "
                "96 (b,h) units head-sharded over the ranks"),
    "c1": (1, 2, 1, 1, 32, 32, 64, None, "fp32",
           "C1 CPU-reference config: B=1 H=2 N=1024 (32,32) untiled fp32"),
}
STACKS = {"wan": 30, "wan_3hw": 30}   # strong-scaled multi-layer workloads (layers per step)


def job_config(name, world, iterations):
    """The ``config`` dict both arms print (identical, so the driver can match them)."""
    B, H, fkv, fq, h, w, d, nb, dt, desc = CONFIGS[name]
    strong = name in STACKS
    if isinstance(nb, tuple) and nb[0] == "aligned":
        plan = f"aligned ({''.join(nb[1])}, rest)"
    elif isinstance(nb, tuple):
        plan = f"neighborhoods {nb[0]}x{nb[1]}x{nb[2]}"
    else:
        plan = {None: "untiled (fh,w)", "mis": "raw (1260,26)"}.get(nb)
    return {"workload": desc, "config": name, "B_per_layer": B, "H": H, "frames_q": fq, "frames_kv": fkv,
            "h": h, "w": w, "d": d, "plan": plan, "iterations": iterations,
            "layers_per_step": STACKS.get(name, world),
            "global_batch": B if strong else B * world,
            "units_per_step": B * H * STACKS.get(name, world),
            "parallelism": f"(b,h) head shards over {world} rank(s), no data-path collective",
            "scaling": "strong" if strong else "weak",
            "l2": "flushed between timed steps (256 MB rewrite, outside events)"}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            j = json.load(fh)
        return {"hbm": j["hbm_gbs"], "tc_burst": j["bf16_tflops"],
                "tc_sustained": j.get("bf16_tflops_sustained", j["bf16_tflops"]), "src": "measured"}
    except Exception:
        return {"hbm": 6650.0, "tc_burst": 1590.0, "tc_sustained": 1400.0, "src": "fallback"}


def workload(name, iterations):
    import paper_2602_12271_b200 as pk

    B, H, fkv, fq, h, w, d, nb, dt, desc = CONFIGS[name]
    shape = pk.VideoShape(fkv, h, w)
    if nb is None:
        plan = pk.aligned_config(shape, ("f", "h"))
        low = pk.lower_square(plan)
    elif nb == "mis":
        plan = pk.config_from_sizes(shape, 1260, 26)
        low = pk.lower_square(plan)
    elif nb[0] == "aligned":
        plan = pk.aligned_config(shape, nb[1])
        low = pk.lower_square(plan)
    else:
        plan = pk.make_tile_plan(shape, pk.aligned_config(shape, ("f", "h")), nb)
        low = pk.lower_chunked(plan, fq) if fq != fkv else pk.lower_square(plan)
    return dict(B=B, H=H, fkv=fkv, fq=fq, h=h, w=w, d=d, dv=d, nb=nb, dtype=dt, desc=desc,
                plan=plan, low=low, T=iterations, nq=fq * h * w, nk=fkv * h * w)


def algorithmic(wl):
    """Per-layer useful FLOPs by stage and compulsory bytes."""
    low, T, d, dv = wl["low"], wl["T"], wl["d"], wl["dv"]
    gq, gk = low.c1_q * low.c2, low.c1_kv * low.c2
    s1, s2 = low.s1, low.s2
    units = wl["B"] * wl["H"]
    eb = 2 if wl["dtype"] == "bf16" else 4
    # row stage (∝ s1 s2^2): beta_R and alpha_L every iteration, Y once
    row = units * gq * gk * s1 * s2 * s2 * 2 * (2 * T * d + dv)
    # column stage: beta_L T times, O once, alpha_R (T-1) times  (∝ s2 s1^2)
    col = units * gq * gk * s2 * s1 * s1 * 2 * (T * d + dv + (T - 1) * d)
    total = row + col
    bytes_ = units * (2 * wl["nq"] * d + wl["nk"] * (d + dv)) * eb
    dense = units * 2 * wl["nq"] * wl["nk"] * (d + dv)
    return dict(row=row, col=col, total=total, bytes=bytes_, dense=dense)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [ln for ln in out.splitlines() if ln.strip()]
            except Exception:
                self.lines = []

    def summary(self):
        sms, maxs, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sms.append(float(parts[0]))
                maxs.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": max(maxs), "reasons": sorted(reasons),
                "samples": len(sms)}


def time_steps(fn, steps, warmup, flush, stream):
    """Sum of per-step CUDA-event times (ms) over `steps` steps, L2 flushed between."""
    import torch

    for _ in range(warmup):
        flush()
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        flush()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs)


def dense_baselines(wl, q, k, v, steps, warmup, flush, stream):
    import torch

    res = {}
    qh, kh, vh = (x.transpose(1, 2).contiguous() for x in (q, k, v))   # (B, N, H, d)

    def sdpa_cudnn():
        from torch.nn.attention import SDPBackend, sdpa_kernel

        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            return torch.nn.functional.scaled_dot_product_attention(q, k, v)

    def sdpa_flash():
        from torch.nn.attention import SDPBackend, sdpa_kernel

        with sdpa_kernel([SDPBackend.FLASH_ATTENTION]):
            return torch.nn.functional.scaled_dot_product_attention(q, k, v)

    def fa2():
        from flash_attn import flash_attn_func

        return flash_attn_func(qh, kh, vh)

    def flashinfer_prefill():
        import flashinfer

        return [flashinfer.single_prefill_with_kv_cache(qh[b], kh[b], vh[b]) for b in range(qh.shape[0])]

    cands = [("torch_sdpa_cudnn", sdpa_cudnn), ("torch_sdpa_flash", sdpa_flash),
             ("flash_attn_2.8", fa2), ("flashinfer_single_prefill", flashinfer_prefill)]
    for name, fn in cands:
        try:
            fn()
            torch.cuda.synchronize()
            ms = time_steps(fn, steps, warmup, flush, stream) / steps
            res[name] = round(ms, 5)
        except Exception as e:   # backend unavailable for this shape/dtype
            res[name] = f"unavailable: {type(e).__name__}: {str(e)[:80]}"
    return res


# --------------------------------------------------------------------------
# reference CPU arm
# --------------------------------------------------------------------------

_CPU = {}   # job description + pre-generated inputs, inherited by the forked pool workers


def _cpu_unit(i):
    """One (b,h) unit through the unmodified reference (or the oracle port); returns seconds.
    Inputs were generated before the pool was forked (outside every timed region)."""
    import numpy as np

    kind, wl = _CPU["kind"], _CPU["wl"]
    q, k, v = _CPU["inputs"][i % len(_CPU["inputs"])]
    T = wl["T"]
    t0 = time.perf_counter()
    if kind == "reference":
        import monarchbench as mb

        shape = mb.VideoShape(wl["fkv"], wl["h"], wl["w"])
        if wl["nb"] is None or wl["nb"][0] == "aligned":
            cfg = mb.aligned_config(shape, ("f", "h") if wl["nb"] is None else wl["nb"][1])
            fac, _ = mb.solve(mb.AttentionProblem(q, k, v, shape), cfg, mb.SolverConfig(iterations=T))
        elif wl["nb"] == "mis":
            cfg = mb.config_from_sizes(shape, 1260, 26)
            fac, _ = mb.solve(mb.AttentionProblem(q, k, v, shape), cfg, mb.SolverConfig(iterations=T))
        else:
            plan = mb.make_tile_plan(shape, mb.aligned_config(shape, ("f", "h")), wl["nb"])
            qq = q
            if wl["fq"] != wl["fkv"]:   # chunked-KV via the square embedding
                qq = np.vstack([np.zeros((wl["nk"] - wl["nq"], wl["d"]), np.float32), q])
            fac, _ = mb.solve_tiled(mb.AttentionProblem(qq, k, v, shape), plan, mb.SolverConfig(iterations=T))
        mb.attention_output(fac, v)
    else:
        from oracle import monarch_oracle as orc

        low = wl["low"]
        oq = np.arange(low.n_q) if low.q_order is None else low.q_order
        ok = np.arange(low.n_kv) if low.kv_order is None else low.kv_order
        orc.forward_phi(q, k, v, oq, ok, low.c1_q, low.c1_kv, low.c2, low.s1, low.s2, T)
    return time.perf_counter() - t0


def _ref_kind():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "monarchbench")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        return "reference"
    return "port"


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


class CpuArm:
    """The reference CPU path on the host cores: inputs generated once, one process
    pool forked once (both outside the timed regions); a timed "wave" runs one unit
    per pool process concurrently."""

    def __init__(self, cfg_name, T, cores):
        import multiprocessing as mp
        import numpy as np

        _env_threads()
        self.kind = _ref_kind()
        self.wl = workload(cfg_name, T)
        self.cores = cores
        self.units = self.wl["B"] * self.wl["H"] * STACKS.get(cfg_name, 1)   # units of one step (1 rank)
        self.wave = min(cores, self.units)
        rng = np.random.default_rng(1000)
        wl = self.wl
        _CPU.update(kind=self.kind, wl=wl, inputs=[
            (rng.standard_normal((wl["nq"], wl["d"])).astype(np.float32),
             rng.standard_normal((wl["nk"], wl["d"])).astype(np.float32),
             rng.standard_normal((wl["nk"], wl["dv"])).astype(np.float32)) for _ in range(min(self.wave, 4))])
        self.pool = mp.get_context("fork").Pool(self.wave) if self.wave > 1 else None

    def wave_s(self):
        """Wall seconds for one wave of `wave` concurrent units."""
        t0 = time.perf_counter()
        if self.pool is not None:
            self.pool.map(_cpu_unit, range(self.wave), chunksize=1)
        else:
            _cpu_unit(0)
        return time.perf_counter() - t0

    def step_ms(self):
        """One step (all `units`) extrapolated from one timed wave: waves run back to back."""
        waves = -(-self.units // self.wave)
        return self.wave_s() * 1e3 * waves, waves

    def serial_unit_ms(self):
        return _cpu_unit(0) * 1e3

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()

    def describe(self, waves):
        full = waves == 1 and self.wave == self.units
        what = (f"full step: {self.units} (b,h) units run concurrently on a pool of {self.wave} processes"
                if full else
                f"one wave of {self.wave} concurrent (b,h) units timed per step, x{waves} waves for the "
                f"step's {self.units} units (extrapolated linearly)")
        return what + "; numpy single-threaded per unit; inputs and pool created outside the timed region"


def _env_threads():
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(var, "1")


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    arm = CpuArm(args.config, args.iters, cores)
    for _ in range(args.warmup):
        arm.wave_s()
    times, waves = [], 1
    for _ in range(args.steps):
        ms, waves = arm.step_ms()
        times.append(ms)
    serial = arm.serial_unit_ms()
    arm.close()
    ms = sum(times) / len(times)
    strong = args.config in STACKS
    value = ms if strong else ms / 1   # one rank's step = one layer (weak) / the whole stack (strong)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3),
        "unit": "ms/stack" if strong else "ms/layer",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic N(0,1) q/k/v (seeded)",
        "config": job_config(args.config, world, args.iters),
        "cpu_baseline": {"value": round(value, 3), "unit": "ms/stack" if strong else "ms/layer", "cores": arm.wave,
                         "kind": arm.kind, "sample": arm.describe(waves), "cpu_model": _cpu_model(),
                         "host_cores": cores, "serial_ms_per_unit_1core": round(serial, 2),
                         "serial_ms_per_step_1core": round(serial * arm.units, 1)},
        "e2e": {"value": round(value, 3), "unit": "ms/stack" if strong else "ms/layer",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

class _Dist:
    """Barrier / max-reduce across ranks: NCCL when every rank has its own GPU, gloo
    (host tensors) when ranks share a device (e.g. --gpus 2 on a one-GPU box)."""

    def __init__(self, world, local):
        import torch
        import torch.distributed as dist

        self.world = world
        self.dist = dist
        ndev = torch.cuda.device_count()
        self.shared = world > ndev
        self.device = torch.device("cuda", local % ndev)
        self.backend = None
        if world > 1:
            self.backend = "gloo" if self.shared else "nccl"
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.device)
            else:
                dist.init_process_group("gloo")

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x):
        import torch

        if self.world == 1:
            return x
        dev = self.device if self.backend == "nccl" else torch.device("cpu")
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.barrier()
            self.dist.destroy_process_group()


def _merge_stages(recs, steps):
    """Per-stage device time per step from per-launch (name, start, ms) records.  Launches of
    one stage that overlap in time (the two concurrent halves on two streams) are merged
    into one span [first start, last end] carrying the whole stage's work; sequential
    launches of a stage (one per refinement) are summed.  Shares and the roofline then
    use whole-stage work over whole-stage time."""
    per_step = len(recs) // max(steps, 1)
    stages = {}
    for sidx in range(steps):
        chunk = recs[sidx * per_step:(sidx + 1) * per_step]
        spans = {}   # name -> list of [lo, hi, launches]
        for name, st, ms in chunk:
            lst = spans.setdefault(name, [])
            for sp in lst:
                if st < sp[1] and st + ms > sp[0]:   # overlaps an open span of this stage
                    sp[0], sp[1], sp[2] = min(sp[0], st), max(sp[1], st + ms), sp[2] + 1
                    break
            else:
                lst.append([st, st + ms, 1])
        for name, lst in spans.items():
            stages.setdefault(name, []).append((sum(hi - lo for lo, hi, _ in lst), sum(n for _, _, n in lst),
                                                len(lst)))
    out = []
    for name, vals in stages.items():
        nv = len(vals)
        out.append({"name": name, "ms_avg": round(sum(v for v, _, _ in vals) / nv, 5),
                    "launches_per_step": sum(n for _, n, _ in vals) / nv,
                    "stage_spans_per_step": sum(k for _, _, k in vals) / nv})
    return out, per_step


def run_ours(args):
    import torch

    import paper_2602_12271_b200 as pk
    from paper_2602_12271_b200 import _lib, ops, shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    D = _Dist(world, local)
    torch.cuda.set_device(D.device)
    dev = D.device
    stream = torch.cuda.current_stream(dev)

    name = args.config
    strong = name in STACKS
    layers = STACKS.get(name, 1)
    wl = workload(name, args.iters)
    dtype = torch.bfloat16 if wl["dtype"] == "bf16" else torch.float32
    B, H = wl["B"], wl["H"]
    # (b,h) units of the job: weak -> `world` layers of B*H units (rank r owns layer r);
    # strong -> one B*H layer split over the ranks (each of the `layers` layers alike)
    if strong:
        start, stop = shard.head_shard(B, H, world, rank)
    else:
        start, stop = shard.head_shard(B * world, H, world, rank)
    spans = [shard.head_shard(B, H, world, r) if strong else shard.head_shard(B * world, H, world, r)
             for r in range(world)]
    units = stop - start
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    # the rank's units as the heads of a size-1 batch (shard.local_slice layout)
    q = torch.randn(1, units, wl["nq"], wl["d"], device=dev, dtype=dtype, generator=g)
    k = torch.randn(1, units, wl["nk"], wl["d"], device=dev, dtype=dtype, generator=g)
    v = torch.randn(1, units, wl["nk"], wl["dv"], device=dev, dtype=dtype, generator=g)
    out = torch.empty(1, units, wl["nq"], wl["dv"], device=dev, dtype=dtype)
    flush_buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def flush():
        flush_buf.zero_()

    low = wl["low"]
    lib = _lib.load()
    prep = ops.prepare(q, k, v, out, low, wl["T"])
    nbytes = lib.mbx_workspace_bytes(prep.desc)
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    path = {0: "simt", 1: "tcgen05"}[lib.mbx_selected_path(prep.desc)]
    import ctypes

    def layer():
        st = lib.mbx_forward(ctypes.byref(prep.desc), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                             out.data_ptr(), None, None, ws.data_ptr(), nbytes, stream.cuda_stream)
        if st != 0:
            _lib.check(st)

    def step():
        for _ in range(layers):
            layer()

    # ---- timed region (device time, max over ranks) ----
    step()
    torch.cuda.synchronize()
    D.barrier()
    with ClockSampler(dev.index) as clk:
        total_ms = time_steps(step, args.steps, args.warmup, flush, stream)
        torch.cuda.synchronize()
    D.barrier()
    total_ms = D.max(total_ms)
    ms_step = total_ms / args.steps
    value = ms_step if strong else ms_step / world   # ms per stack (strong) / whole-job ms per layer (weak)
    ms_layer_local = ms_step / layers                # this rank's device time for one layer of its units

    # ---- per-kernel shares (same stream, L2 flushed, CUDA events per launch) ----
    prof_steps = max(3, min(args.steps, 20))
    lib.mbx_profile_enable(1)
    for _ in range(prof_steps):
        flush()
        layer()
    torch.cuda.synchronize()
    lib.mbx_profile_enable(0)
    recs = _lib.profile_collect_ex()
    kernels, launches_per_layer = _merge_stages(recs, prof_steps)
    alg = algorithmic(wl)
    alg_local = {kk: vv * units / (B * H) for kk, vv in alg.items()}   # this rank's share of one layer
    peaks = _peaks()
    ksum = sum(kk["ms_avg"] for kk in kernels) or ms_layer_local
    for kk in kernels:
        kk["share"] = round(kk["ms_avg"] / ksum, 4)
    dom = max(kernels, key=lambda kk: kk["ms_avg"]) if kernels else None
    roofline = None
    eb = 2 if dtype == torch.bfloat16 else 4
    if dom is not None:
        kname = dom["name"]
        if "row" in kname:
            flops = alg_local["row"]
            byts = units * (wl["nq"] * wl["d"] + wl["nk"] * (wl["d"] + wl["dv"])) * eb
        elif "column" in kname:
            flops = alg_local["col"]
            byts = units * (wl["nq"] * (wl["d"] + wl["dv"])) * eb
        else:
            flops, byts = alg_local["total"], alg_local["bytes"]
        per_launch_spans = 1
        t_s = dom["ms_avg"] * 1e-3
        t_tc = flops / (peaks["tc_burst"] * 1e12)
        t_hbm = byts / (peaks["hbm"] * 1e9)
        if t_tc >= t_hbm:
            ach = flops / t_s / 1e12
            roofline = {"bound": "tensor", "achieved": round(ach, 2), "peak": peaks["tc_burst"],
                        "unit": "TFLOP/s", "frac": round(ach / peaks["tc_burst"], 4)}
        else:
            ach = byts / t_s / 1e9
            roofline = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm"],
                        "unit": "GB/s", "frac": round(ach / peaks["hbm"], 4)}
        # The two-stage design moves the [aL | Y] exchange (SURVEY.md §8d "intermediate
        # materialisation") through L2: bytes including it, against the measured L2 read
        # bandwidth for working sets beyond 48 MB (scripts/microbench.cu,
        # profiles/r1_microbench_memory.json) -- the bound the stages actually run into.
        if wl["T"] == 1 and ("row" in kname or "column" in kname):
            exch = units * (low.c1_q * low.c2) * (low.c1_kv * low.c2) * low.s1 * low.s2 * ((wl["d"] + wl["dv"]) * eb + 4)
            l2b = byts + exch
            l2_peak = _l2_peak()
            if l2_peak:
                roofline["exchange_l2"] = {"bytes_per_launch": int(l2b), "achieved": round(l2b / t_s / 1e9, 1),
                                           "peak": l2_peak, "unit": "GB/s", "frac": round(l2b / t_s / 1e9 / l2_peak, 4),
                                           "peak_source": "L2 read GB/s, >= 48 MB working set, profiles/r1_microbench_memory.json"}
        roofline.update({"kernel": kname, "traffic": _ncu_traffic(kname, name),
                         "peak_source": f"{peaks['src']} (MEASURED_PEAKS.json burst)",
                         "algorithmic_flops_per_launch": int(flops), "algorithmic_bytes_per_launch": int(byts),
                         "launches_merged": dom["launches_per_step"], "spans": per_launch_spans})

    # ---- eager per-call latency through the public API (device tensors, no L2 flush) ----
    eager = None
    if not strong:
        plan = wl["plan"]
        kvf = wl["fkv"] if wl["fq"] != wl["fkv"] else None
        o2 = torch.empty_like(out)
        for _ in range(5):
            pk.monarch_attention(q, k, v, plan, iterations=wl["T"], kv_frames=kvf, out=o2)
        torch.cuda.synchronize()
        n_calls = 200
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(n_calls):
            pk.monarch_attention(q, k, v, plan, iterations=wl["T"], kv_frames=kvf, out=o2)
        t1 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        dev_ms = e0.elapsed_time(e1) / n_calls
        eager = {"host_enqueue_us_per_call": round((t1 - t0) * 1e6 / n_calls, 2),
                 "wall_us_per_call": round((t2 - t0) * 1e6 / n_calls, 2),
                 "device_us_per_call_hot_l2": round(dev_ms * 1e3, 2),
                 "overhead_us_above_device": round(max(0.0, (t2 - t0) * 1e6 / n_calls - dev_ms * 1e3), 2),
                 "calls": n_calls, "api": "paper_2602_12271_b200.monarch_attention (device tensors)"}

    # ---- backward pass (finetuning step): forward recompute with factor export + mbx_backward ----
    bwd = None
    if not strong and not args.no_backward:
        dout = torch.randn(out.shape, device=dev, dtype=dtype, generator=g)

        def bwd_step():
            ops.backward(q, k, v, dout, low, wl["T"])

        bwd_step()
        torch.cuda.synchronize()
        bsteps = max(3, min(args.steps, 10))
        bwd_ms = D.max(time_steps(bwd_step, bsteps, 2, flush, stream)) / bsteps
        lib.mbx_profile_enable(1)
        flush()
        bwd_step()
        torch.cuda.synchronize()
        lib.mbx_profile_enable(0)
        brecs = _lib.profile_collect_ex()
        bk = {}
        for nm, _, ms in brecs:
            bk[nm] = bk.get(nm, 0.0) + ms
        dense_bwd = None
        if rank == 0 and not args.no_dense:
            try:
                from torch.nn.attention import SDPBackend, sdpa_kernel

                qd, kd, vd = (x.detach().clone().requires_grad_(True) for x in (q, k, v))

                def dense_bwd_step():
                    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
                        o_ = torch.nn.functional.scaled_dot_product_attention(qd, kd, vd)
                    o_.backward(dout)

                dense_bwd_step()
                torch.cuda.synchronize()
                dense_bwd = round(time_steps(dense_bwd_step, bsteps, 2, flush, stream) / bsteps, 5)
            except Exception as e:   # backend unavailable
                dense_bwd = f"unavailable: {type(e).__name__}"
        bwd = {"ms": round(bwd_ms, 5), "includes": "forward recompute with factor export + mbx_backward",
               "dense_fwd_plus_bwd_ms_cudnn": dense_bwd,
               "arith": ("TF32 tensor-core batched GEMMs (in-library mma.sync kernel; cuBLAS for 5 contractions) + fp32 softmax-backward kernels" if dtype == torch.bfloat16
                         else "fp32 SIMT (batched GEMM chain)"),
               "kernels_ms": {kk: round(vv, 5) for kk, vv in sorted(bk.items(), key=lambda x: -x[1])[:8]}}

    # ---- end-to-end through the public API with host buffers ----
    # monarch_attention_host: pinned host q/k/v in, host output back, H2D / forward / D2H
    # pipelined over (b,h) chunks (all inside the timed region), once per layer of the step
    pin = [x.cpu().pin_memory() for x in (q, k, v)]
    out_h = torch.empty(out.shape, dtype=dtype).pin_memory()
    plan = wl["plan"]
    kvf = wl["fkv"] if wl["fq"] != wl["fkv"] else None

    def e2e_step():
        for _ in range(layers):
            pk.monarch_attention_host(pin[0], pin[1], pin[2], plan, iterations=wl["T"], kv_frames=kvf, out=out_h)

    e2e_steps = args.steps if not strong else max(3, min(args.steps, 5))
    D.barrier()
    e2e_total = D.max(time_steps(e2e_step, e2e_steps, min(args.warmup, 3), flush, stream))
    e2e_ms = e2e_total / e2e_steps
    e2e_value = e2e_ms if strong else e2e_ms / world
    h2d = sum(x.numel() for x in pin) * eb * layers
    d2h = out_h.numel() * eb * layers

    # ---- optional NCCL all-gather of the output shards (sequence-parallel DiT block) ----
    allgather = None
    if strong and world > 1 and D.backend == "nccl":
        def gather_step():
            for _ in range(layers):
                shard.all_gather_heads(out, B, H)

        gather_step()
        torch.cuda.synchronize()
        D.barrier()
        ag = D.max(time_steps(gather_step, max(3, min(args.steps, 10)), 2, flush, stream))
        ag_steps = max(3, min(args.steps, 10))
        allgather = {"ms_per_step": round(ag / ag_steps, 4), "ms_per_layer": round(ag / ag_steps / layers, 4),
                     "bytes_per_rank_per_layer": int(out.numel() * eb), "backend": "nccl",
                     "communicator_size": world}

    # ---- dense attention on the same (local) shape ----
    dense = {}
    if not args.no_dense and rank == 0:
        dense = dense_baselines(wl, q, k, v, max(3, min(args.steps, 20)), args.warmup, flush, stream)
    dense_nums = {kname: val for kname, val in dense.items() if isinstance(val, float)}
    best_dense = min(dense_nums.values()) if dense_nums else None   # ms per layer of the local units

    # ---- CPU baseline (rank 0, N=1 only; bounded sample) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = len(os.sched_getaffinity(0))
        arm = CpuArm(name, wl["T"], cores)
        arm.wave_s()   # warm-up (imports, page faults)
        ms_cpu, waves = arm.step_ms()
        serial = arm.serial_unit_ms()
        arm.close()
        cpu = {"value": round(ms_cpu, 2), "unit": "ms/stack" if strong else "ms/layer", "cores": arm.wave,
               "kind": arm.kind, "sample": arm.describe(waves), "cpu_model": _cpu_model(), "host_cores": cores,
               "serial_ms_per_unit_1core": round(serial, 2), "serial_ms_per_step_1core": round(serial * arm.units, 1)}

    if rank == 0:
        unit = "ms/stack" if strong else "ms/layer"
        line = {
            "metric": METRIC, "value": round(value, 5), "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": False, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": wl["dtype"], "data": "synthetic N(0,1) q/k/v generated on device (seeded)",
            "config": job_config(name, world, wl["T"]),
            "shards": {"units_per_rank": [b_ - a_ for a_, b_ in spans], "rank_spans": spans,
                       "backend": D.backend, "shared_gpu": D.shared, "path": path,
                       "plan": plan.descriptor() if hasattr(plan, "descriptor") else str(plan)},
            "dense_fa_ms": dense, "dense_fa_best_ms": best_dense,
            "speedup_vs_dense": round(best_dense / ms_layer_local, 3) if best_dense else None,
            "effective_tflops": round(alg_local["total"] / (ms_layer_local * 1e-3) / 1e12 * world, 2),
            "tc_util": round(alg_local["total"] / (ms_layer_local * 1e-3) / 1e12 / peaks["tc_burst"], 4),
            "algorithmic": {"flops_per_layer": alg["total"], "bytes_per_layer": alg["bytes"],
                            "dense_flops_per_layer": alg["dense"], "rank0_units": units},
            "kernels": kernels, "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 5), "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "paper_2602_12271_b200.monarch_attention_host"},
            "eager": eager, "allgather": allgather, "backward": bwd,
            "gpu_launches": int(round(launches_per_layer * layers * args.steps)),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    D.close()


def _self_launch(args):
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def _l2_peak():
    """Measured L2 read bandwidth (GB/s) for working sets beyond the L2-resident sweet spot."""
    p = os.path.join(ROOT, "profiles", "r1_microbench_memory.json")
    try:
        with open(p) as fh:
            rd = json.load(fh)["l2_read_GBps"]
        return float(min(v for kk, v in rd.items() if int(kk) >= 48))
    except Exception:
        return None


def _ncu_traffic(kernel, config):
    """dram bytes per launch of `kernel` from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            j = json.load(fh)
        return j.get(config, {}).get(kernel)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="sf", choices=sorted(CONFIGS))
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-backward", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _self_launch(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
