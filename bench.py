#!/usr/bin/env python3
"""Benchmark: INT3+LoRC MoE-layer latency (us) & achieved HBM GB/s on B200.

Default workload (BASELINE.json configs[1]): one Mixtral-8x7B MoE layer —
8 experts (d=4096, f=14336), top-2 router, INT3 g64 asymmetric weights with
ragged symm-int3 compensator ranks — at batch 1 (decode), random-init
synthetic weights/activations of that shape.  A "step" is one full layer
call: router top-k -> permute -> grouped W3A16+LoRC (w1|w3 + SwiGLU) ->
grouped W3A16+LoRC (w2) -> weighted combine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl milo|reference]
                    [--config mixtral|deepseek|arctic] [--batch M] [--no-sweep]

Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events on
the launching stream; the L2 flush (256 MiB write + 256 MiB read) between steps is outside the
events.  Barrier + synchronize around the timed region, max over ranks.
`value` = mean layer latency (us, lower is better).  `e2e` = the same through
the host-buffer C-ABI entry point (milo_moe_forward_host: pinned host x and
logits copied in, output copied back inside the timed call), wall clock.
`roofline` = the dominant kernel (grouped GEMM phase 1, w1|w3 + SwiGLU),
algorithmic bytes (matrix_memory_bytes of every touched expert + fp16
activations) / its CUDA-event duration, against the
measured HBM copy bandwidth in MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "INT3+LoRC MoE-layer latency (us) & achieved HBM GB/s, batch 1-256, 1/8 GPU"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - sampling is best effort
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                sm = self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM)
                rs = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((sm, rs))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        busy = [s for s in self.samples if not (s[1] & 0x1)] or self.samples
        reasons = set()
        for _, r in busy:
            for bit, name in self.REASONS.items():
                if r & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": float(np.median([s[0] for s in busy])), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_inputs(spec, m, n_steps, seed):
    """The synthetic per-step inputs both arms use: x (binary16 values, as the
    kernels and gemm.cpp:144-146 round them) and fp32 router logits."""
    rng = np.random.default_rng(seed)
    xs = [rng.normal(0, 1, (m, spec.d)).astype(np.float16) for _ in range(n_steps)]
    ls = [rng.normal(0, 1, (m, spec.experts)).astype(np.float32) for _ in range(n_steps)]
    return xs, ls


def input_seed(args, m, rank=0):
    return args.seed * 1000 + m * 16 + rank


class CpuReference:
    """The reference CPU implementation of the layer on the host cores: the
    compiled reference's gemm_w3a16 (oracle/_ref) composed per expert, every
    (expert, matrix, column slice) call through its parallel_for over all
    threads (oracle/ref/ref_capi.cpp); our C restatement if oracle/_ref is
    missing.  Weights are copied in and sliced once, outside any timing."""

    def __init__(self, spec, routed, shared):
        from oracle.oracle import Comp, Oracle, Packed, RefMoE
        self.kind = "reference" if Oracle.available("ref") else "port"
        self.cores = os.cpu_count() or 1
        self.spec = spec
        self.orc = Oracle("oracle")

        def cv(P):
            return Packed(P.rows, P.cols, 0, False, P.mode, 64, P.words, None, None, P.scales, P.zeros)

        def cc(c):
            if c is None:
                return None
            return Comp(c.rows, c.cols, c.rank, 1, None, None, c.qu_codes, c.qu_scales, c.qvt_codes,
                        c.qvt_scales, 64)

        self.ex = [{"w": [cv(P) for P in h.w], "c": [cc(c) for c in h.c]} for h in routed]
        self.sh = [{"w": [cv(P) for P in h.w], "c": [cc(c) for c in h.c]} for h in shared]
        self.h = RefMoE(Oracle("ref"), self.ex, self.sh, self.cores) if self.kind == "reference" else None

    def forward(self, x, logits):
        """One layer call (router + experts + combine) on the host; fp32 out."""
        ids, w = self.orc.router_topk(logits, self.spec.top_k, self.spec.score_mode)
        x = np.asarray(x, np.float32)
        if self.h is not None:
            return self.h.forward(x, ids, w), ids
        return self.orc.moe_forward(self.ex, self.sh, x, ids, w, n_threads=self.cores), ids

    def time(self, xs, ls):
        times = []
        for x, lg in zip(xs, ls):
            t0 = time.perf_counter()
            self.forward(x, lg)
            times.append(time.perf_counter() - t0)
        return float(np.mean(times)) * 1e6

    def describe(self, steps, m):
        how = ("the reference's gemm_w3a16 (oracle/_ref)" if self.kind == "reference"
               else "the C restatement (oracle/milo_oracle.c)")
        return (f"{steps} x {self.spec.name} layer calls at batch {m}: {how} per (touched expert, "
                f"matrix, 128-column slice) through parallel_for on {self.cores} threads "
                f"({cpu_model()}); weights resident in host RAM")


def rank_summary(spec):
    """The compensator ranks of the benchmarked layer: the frozen plan's policy and
    per-matrix ranks (w1, w3, w2 per expert), else the config's rank vector."""
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from paper_2504_02658_b200.synth import expert_ranks, load_rank_plan
    plan = load_rank_plan(spec)
    if plan is None:
        return {"routed": list(spec.routed_ranks), "shared": spec.rank_shared}
    routed = [expert_ranks(spec, e, plan) for e in range(spec.experts)]
    flat = [r for t in routed for r in t]
    out = {"plan": f"{spec.plan}.plan.json ({plan.policy}, the reference's plan_ranks; "
                   "tools/make_rank_plans.py)", "avg_routed": round(float(np.mean(flat)), 2),
           "min_routed": int(min(flat)), "max_routed": int(max(flat))}
    if spec.experts <= 8:
        out["routed_w1_w3_w2"] = routed
    if spec.shared:
        out["shared"] = [plan.ranks[f"layer0.shared_expert{s}.{w}"] for s in range(spec.shared)
                         for w in ("w1", "w3", "w2")]
    return out


def config_dict(spec, m, parallelism):
    return {"workload": spec.name, "batch": m, "experts": spec.experts, "top_k": spec.top_k,
            "d": spec.d, "f": spec.f, "shared_experts": spec.shared,
            "ranks": rank_summary(spec),
            "parallelism": parallelism, "tokens_per_rank": m,
            "inputs": "numpy default_rng(seed*1000 + 16 m + rank): x N(0,1) as binary16, logits N(0,1) f32",
            "l2": "flushed between steps (256 MiB write + 256 MiB read, outside the timed events)"}


def run_reference_arm(args, spec):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2504_02658_b200.synth import build_host_layer
    routed, shared = build_host_layer(spec, seed=args.seed)
    cpu = CpuReference(spec, routed, shared)
    steps = max(1, args.steps)
    m = args.batch
    xs, ls = host_inputs(spec, m, args.warmup + steps, input_seed(args, m))
    for i in range(min(args.warmup, 1)):
        cpu.forward(xs[i], ls[i])
    us = cpu.time(xs[args.warmup:], ls[args.warmup:])
    line = {
        "impl": "reference", "metric": METRIC, "value": round(us, 1), "unit": "us",
        "n_gpus": ws, "steps": steps, "warmup": args.warmup, "ms_per_step": round(us / 1e3, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f16 (activations, de-quantized weights) / f32 accumulate",
        "data": "synthetic (random-init INT3 g64 weights, symm-int3 LoRC, N(0,1) activations "
                "and router logits)",
        "config": config_dict(spec, m, "ep%d" % ws if ws > 1 else "single GPU"),
        "cpu_baseline": {"value": round(us, 1), "unit": "us", "cores": cpu.cores, "kind": cpu.kind,
                         "sample": cpu.describe(steps, m)},
        "e2e": {"value": round(us, 1), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="milo", choices=["milo", "reference"])
    ap.add_argument("--config", default="mixtral", choices=["mixtral", "deepseek", "arctic"])
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline timing")
    ap.add_argument("--no-parity", action="store_true", help="skip the reference parity check")
    ap.add_argument("--ep", action="store_true", help="expert-parallel layer (default when N > 1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2504_02658_b200.synth import CONFIGS
    spec = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, spec)

    import torch
    import torch.distributed as dist
    import paper_2504_02658_b200 as mb
    from paper_2504_02658_b200.synth import build_host_layer, layer_traffic

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    mb.device_check()
    peaks, peaks_src = load_peaks()

    routed_h, shared_h = build_host_layer(spec, seed=args.seed)

    def dev_expert(h):
        return mb.Expert(*(mb.Weight(P) for P in h.w), *((mb.Comp(c) if c is not None else None) for c in h.c))

    shared = [dev_expert(h) for h in shared_h]
    use_ep = ws > 1 or args.ep
    if use_ep and ws == 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
    if use_ep:
        # expert parallel: rank r owns experts [r E / N, (r + 1) E / N),
        # tokens move over NCCL all-to-all-v; m tokens per rank (weak scaling)
        # the C++ layer over NCCL: router, dispatch, grouped ncclSend / ncclRecv exchanges,
        # owned experts, shared experts and combine in one stream-ordered call
        from paper_2504_02658_b200.ep import NativeEPLayer
        per = (spec.experts + ws - 1) // ws
        owned = [dev_expert(h) for h in routed_h[rank * per:(rank + 1) * per]]
        layer = NativeEPLayer(owned, shared, spec.experts, spec.top_k, spec.score_mode)
        layer.capacity = 0  # every rank runs the same batch (weak scaling by tokens): C = m K
    else:
        experts = [dev_expert(h) for h in routed_h]
        layer = mb.MoELayer(experts, shared, top_k=spec.top_k, score_mode=spec.score_mode)

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    flush_r = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")

    def flush_l2():
        # write a buffer larger than L2 (126 MB), then read another one so the L2 holds
        # clean lines: the timed layer neither finds its inputs in L2 nor pays for
        # writing back the flush's dirty lines (which a real decode step would not).
        flush.zero_()
        torch.sum(flush_r)
    stream = torch.cuda.current_stream()

    def make_inputs(m, n_steps):
        hx, hl = host_inputs(spec, m, n_steps, input_seed(args, m, rank))
        return [torch.from_numpy(x).cuda() for x in hx], [torch.from_numpy(lg).cuda() for lg in hl], hx, hl

    def time_steps(m, n_steps, warmup, profile=False, keep_first=False):
        xs, ls, hx, hl = make_inputs(m, warmup + n_steps)
        keep = []  # same allocation pattern as the timed loop (outputs kept alive)
        for i in range(warmup):
            keep.append(layer.forward(xs[i], ls[i], return_routing=True))
        del keep
        ids_all = []
        first = None
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(n_steps)]
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = mb.launch_count()
        if profile:
            mb.profile_enable(True)
        # a short device backlog so a host-side hiccup (allocator growth, GC) between
        # two events cannot leave the GPU idle inside a timed step; the host path
        # itself is what the e2e leg measures
        torch.cuda._sleep(2_000_000)
        for i in range(n_steps):
            flush_l2()
            s, e = evs[i]
            s.record(stream)
            if use_ep:  # routing ids for the byte accounting are taken outside the events
                o = layer.forward(xs[warmup + i], ls[warmup + i])
                e.record(stream)
                ids = mb.router_topk(ls[warmup + i], spec.top_k, spec.score_mode)[0]
            else:
                o, ids, _ = layer.forward(xs[warmup + i], ls[warmup + i], return_routing=True)
                e.record(stream)
            ids_all.append(ids)
            if keep_first and i == 0:
                first = (o, hx[warmup], hl[warmup])
        torch.cuda.synchronize()
        if profile:
            mb.profile_enable(False)
        launches = mb.launch_count() - l0
        if ws > 1:
            dist.barrier()
        ms = np.array([s.elapsed_time(e) for s, e in evs])
        ids_np = [i.cpu().numpy() for i in ids_all]
        if keep_first:
            return ms, ids_np, launches, (first[0].cpu().numpy(), first[1], first[2])
        return ms, ids_np, launches

    # ---------------- headline timed region ----------------
    m = args.batch
    with ClockSampler(local) as clk:
        ms, ids_np, launches, first_step = time_steps(m, args.steps, args.warmup, keep_first=True)
    mean_ms = float(ms.mean())
    if ws > 1:
        t = torch.tensor([mean_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        mean_ms = float(t.item())
    traffic = [layer_traffic(spec, routed_h, shared_h, i) for i in ids_np]
    tot_bytes = float(np.mean([t["total_bytes"] for t in traffic]))
    tot_flops = float(np.mean([t["total_flops"] for t in traffic]))

    # ---------------- roofline of the dominant kernel (live CUDA events) ----------------
    ms_p, ids_p, _ = time_steps(m, args.steps, 2, profile=True)
    n1, t1 = mb.profile_read(0)
    n2, t2 = mb.profile_read(1)
    nl, tl = mb.profile_read(2)
    tr_p = [layer_traffic(spec, routed_h, shared_h, i) for i in ids_p]
    p1_bytes = float(np.mean([t["phase1_bytes"] for t in tr_p]))
    p2_bytes = float(np.mean([t["phase2_bytes"] for t in tr_p]))
    hbm = float(peaks["hbm_gbs"])
    single = n2 == 0  # one-launch decode kernel: the whole layer is one kernel
    prefill = m > 64  # tcgen05 path: pf_gemm_kernel<2> (w1|w3) then pf_gemm_kernel<1> (w2)
    bound, unit, peak = "hbm", "GB/s", hbm
    if single:
        dom_bytes = p1_bytes + p2_bytes
        dom_ms = t1 / max(n1, 1)
        dom_name = ("decode_kernel<%d,2,MoE> (whole layer: routing, LoRC, w1|w3+SwiGLU, w2, combine)"
                    % (1 if m <= 8 else 2))
    elif prefill:
        dom_bytes = p1_bytes
        dom_ms = t1 / max(n1, 1)
        dom_name = "pf_gemm_kernel<2,1> (phase 1: w1|w3 + LoRC stages + SwiGLU, tcgen05)"
        bound, unit, peak = "tensor", "TFLOP/s", float(peaks["bf16_tflops"])
    else:
        dom_bytes = p1_bytes
        dom_ms = t1 / max(n1, 1)
        dom_name = "gemv_w3a16_kernel<NT,2> (phase 1: w1|w3 + SwiGLU + LoRC)"
    p1_ms = dom_ms
    p2_ms = t2 / max(n2, 1)
    if dom_ms <= 0:
        achieved = 0.0
    elif bound == "tensor":  # phase-1 flops: 2 matrices of d x f per routed token + LoRC
        p1_flops = float(np.mean([t.get("phase1_flops", 0.0) for t in tr_p]))
        achieved = p1_flops / (dom_ms * 1e-3) / 1e12
    else:
        achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic_ncu = None
    ncu_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(ncu_path):
        try:
            traffic_ncu = json.load(open(ncu_path)).get(args.config, {}).get(str(m))
        except Exception:  # noqa: BLE001
            traffic_ncu = None

    # ---------------- end to end through the host-buffer C ABI ----------------
    e2e_steps = max(3, min(args.steps, 50))
    xh = torch.randn(m, spec.d).pin_memory()
    lh = torch.randn(m, spec.experts).pin_memory()
    xn, ln = xh.numpy(), lh.numpy()
    for _ in range(2):
        layer.forward_host(xn, ln)
    if ws > 1:
        dist.barrier()
    wall = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        layer.forward_host(xn, ln)
        wall.append(time.perf_counter() - t0)
    e2e_us = float(np.mean(wall)) * 1e6
    if ws > 1:
        t = torch.tensor([e2e_us], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_us = float(t.item())

    # ---------------- configs[0]: the single 4096 x 14336 linear, r = 32 (N=1) ----------------
    c1 = []
    if not args.no_sweep and ws == 1 and args.config == "mixtral":
        from paper_2504_02658_b200.pack import random_compensator
        from paper_2504_02658_b200.synth import matrix_memory_bytes, packed_random_words
        rng1 = np.random.default_rng(args.seed + 4242)
        k1, n1, r1 = 4096, 14336, 32
        W1 = mb.Weight(packed_random_words(k1, n1, rng1))
        C1 = mb.Comp(random_compensator(k1, n1, r1, rng1))
        for mm in (1, 16, 64, 256):
            A1 = torch.from_numpy(np.random.default_rng(mm).normal(0, 1, (mm, k1)).astype(np.float16)).cuda()
            o1 = torch.empty(mm, n1, device="cuda", dtype=torch.float32)
            for _ in range(3):
                mb.gemm_w3a16(A1, W1, C1, out=o1)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            torch.cuda.synchronize()
            for s_, e_ in ev:
                flush_l2()
                s_.record(stream)
                mb.gemm_w3a16(A1, W1, C1, out=o1)
                e_.record(stream)
            torch.cuda.synchronize()
            us = float(np.mean([s_.elapsed_time(e_) for s_, e_ in ev])) * 1e3
            b = matrix_memory_bytes(k1, n1, r1) + 2 * mm * k1 + 4 * mm * n1
            fl = 2 * mm * k1 * n1 + 2 * mm * r1 * (k1 + n1)
            t_roof = max(b / (hbm * 1e9), fl / (float(peaks["bf16_tflops"]) * 1e12)) * 1e6
            c1.append({"batch": mm, "us": round(us, 2), "GBps": round(b / us / 1e3, 1),
                       "TFLOPs": round(fl / us / 1e6, 2), "roofline_us": round(t_roof, 2),
                       "roofline_frac": round(t_roof / us, 3),
                       "kernel": "decode_kernel (mma.sync)" if mm <= 16 else "pf_gemm_kernel (tcgen05)"})
        del W1, C1

    # ---------------- batch sweep (N=1) ----------------
    sweep = []
    if not args.no_sweep and ws == 1:
        for mm in (1, 16, 64, 256):
            sms, sids, _ = time_steps(mm, 10, 3)
            if os.environ.get("MILO_BENCH_DUMP_STEPS"):
                print(f"sweep m={mm} step ms: " + " ".join(f"{v:.3f}" for v in sms), file=sys.stderr)
            tr = [layer_traffic(spec, routed_h, shared_h, i) for i in sids]
            b = float(np.mean([t["total_bytes"] for t in tr]))
            fl = float(np.mean([t["total_flops"] for t in tr]))
            us = float(sms.mean()) * 1e3
            t_roof = max(b / (hbm * 1e9), fl / (float(peaks["bf16_tflops"]) * 1e12)) * 1e6
            sweep.append({"batch": mm, "us": round(us, 2), "GBps": round(b / us / 1e3, 1),
                          "TFLOPs": round(fl / us / 1e6, 2), "roofline_us": round(t_roof, 2),
                          "roofline_frac": round(t_roof / us, 3)})

    # ---------------- CPU reference: parity of a timed step + baseline (rank 0) ----------------
    cpu = parity = None
    if rank == 0 and not args.no_parity:
        try:
            ref = CpuReference(spec, routed_h, shared_h)
            got, hx0, hl0 = first_step
            want, ref_ids = ref.forward(hx0, hl0)
            den = float(np.sqrt((want.astype(np.float64) ** 2).sum()))
            parity = {"rel_err": float(np.sqrt(((got.astype(np.float64) - want) ** 2).sum()) / den),
                      "ids_equal": bool(np.array_equal(ids_np[0], ref_ids)), "tol": 2.5e-4,
                      "against": ref.kind, "step": "first timed step (same x / logits, fp32 out)"}
            if ws == 1 and not args.no_cpu:
                cpu_steps = 3
                hx, hl = host_inputs(spec, m, cpu_steps, input_seed(args, m) + 7)
                us = ref.time(hx, hl)
                cpu = {"value": round(us, 1), "unit": "us", "cores": ref.cores, "kind": ref.kind,
                       "sample": ref.describe(cpu_steps, m)}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "us", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"unavailable: {exc}"}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    value_us = mean_ms * 1e3
    line = {
        "metric": METRIC, "value": round(value_us, 2), "unit": "us", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(mean_ms, 4),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f16 (activations, de-quantized weights) / f32 accumulate",
        "data": "synthetic (random-init INT3 g64 weights, symm-int3 LoRC, N(0,1) activations "
                "and router logits)",
        "config": config_dict(spec, m, f"ep{ws}" if use_ep else "single GPU"),
        "achieved_GBps_layer": round(tot_bytes / (value_us * 1e-6) / 1e9, 1),
        "layer_bytes": int(tot_bytes), "layer_flops": int(tot_flops),
        "roofline": {"bound": bound, "kernel": dom_name, "achieved": round(achieved, 1), "peak": peak,
                     "unit": unit, "frac": round(achieved / peak, 4), "traffic": traffic_ncu if bound == "hbm" else None,
                     "algorithmic_bytes_per_launch": int(dom_bytes),
                     "launch_us": round(p1_ms * 1e3, 2), "peak_source": peaks_src,
                     "phase2": {"algorithmic_bytes_per_launch": int(p2_bytes),
                                "launch_us": round(p2_ms * 1e3, 2),
                                "achieved": round(p2_bytes / (p2_ms * 1e-3) / 1e9, 1) if p2_ms > 0 else None},
                     "lorc_us_per_step": round(tl / max(1, len(ms_p)) * 1e3, 2),
                     "layer_frac": round(tot_bytes / (value_us * 1e-6) / 1e9 / hbm, 4)},
        "e2e": {"value": round(e2e_us, 2), "unit": "us",
                "h2d_bytes_per_step": int(m * spec.d * 4 + m * spec.experts * 4),
                "d2h_bytes_per_step": int(m * spec.d * 4)},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "parity": parity,
        "sweep": sweep,
        "c1_linear": {"workload": "configs[0]: single INT3 linear 4096x14336, g64, rank-32 LoRC, fp32 out",
                      "sweep": c1} if c1 else None,
    }
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
