#!/usr/bin/env python
"""Benchmark of the B200 VQMC Max-Cut training step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[4], the headline): Max-Cut on a random 3-regular graph with
N = 10,000 vertices, MADE with h = round(5 ln^2 N) = 424, exact autoregressive sampling,
1024 samples per GPU per step, REINFORCE gradient, NCCL all-reduce (N > 1), Adam.
A step is one full VQMC iteration (vqmc::train's worker_body).  Synthetic graph and
random-init weights (no datasets exist for this problem).

Under torchrun (N > 1) every rank drives one GPU; data parallel, weak scaling (1024 samples
per GPU), one NCCL all-reduce of the gradient per step inside the fused step.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=10000)
    ap.add_argument("--graph", choices=["regular3", "maxcut"], default="regular3")
    ap.add_argument("--minibatch", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the bounded CPU sample")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks / e2e / cpu)")
    ap.add_argument("--no-sr", action="store_true", help="skip the SGD + SR step measurement")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Dist:
    """torch.distributed (gloo) for plumbing: id broadcast, barriers, max over ranks."""

    def __init__(self, world, rank):
        self.world, self.rank = world, rank
        self.pg = None
        if world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=rank, world_size=world)
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def bcast_bytes(self, b: bytes) -> bytes:
        if self.world == 1:
            return b
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", "clocks.csv")
        self.nvml = None

    # NVML sampler (every 2 ms in a thread, so even a few-ms timed region is covered); nvidia-smi
    # (-lms 100) is the fallback.
    def _nvml_loop(self):
        import pynvml as nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self._samples.append((sm, mx, rs))
            except Exception:
                pass
            self._first.set()
            self._stop.wait(0.002)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            idx = int(os.environ.get("LOCAL_RANK", "0"))
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                idx = int(vis.split(",")[idx])
            self._h = nv.nvmlDeviceGetHandleByIndex(idx)
            self._samples, self._stop, self._first = [], threading.Event(), threading.Event()
            self._t = threading.Thread(target=self._nvml_loop, daemon=True)
            self._t.start()
            self._first.wait(1.0)
            self.nvml = nv
            return
        except Exception:
            self.nvml = None
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.nvml is not None:
            nv = self.nvml
            self._stop.set()
            self._t.join(timeout=2)
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}
            if not self._samples:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
            reasons = sorted({nm for (_, _, r) in self._samples for nm, b in bits.items() if r & b})
            return {"sm_mhz": float(np.median([x[0] for x in self._samples])),
                    "sm_max_mhz": float(max(x[1] for x in self._samples)), "reasons": reasons,
                    "samples": len(self._samples), "source": "nvml (2 ms)"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def make_instance(args):
    from paper_2106_13308_b200 import api
    if args.graph == "regular3":
        g = api.random_regular_graph(args.n, 3, args.seed)
        desc = f"random 3-regular, |E|={len(g.edges)}"
    else:
        g = api.random_maxcut_graph(args.n, args.seed)
        desc = f"reference G(n,3/4), |E|={len(g.edges)}"
    return g, desc


# ---------------------------------------------------------------------------
# Algorithmic work per kernel launch: FLOPs for the GEMM-shaped
# kernels (tensor-core bound), bytes for the streaming ones (HBM bound).
# ---------------------------------------------------------------------------
def kernel_work(name, n, h, Hd, B, E):
    nnzM2_tail = (n - Hd) * h
    if name in ("z2_tail_sample", "z2_tail_umma"):
        return "tensor", 2.0 * B * nnzM2_tail, "FLOP"
    if name in ("bw_dg1", "bw_dg1_umma"):
        return "tensor", 2.0 * B * n * h, "FLOP"
    if name in ("bw_gw2", "bw_gw2_umma"):
        return "tensor", 2.0 * B * n * (h + 1), "FLOP"
    if name in ("bw_gw1", "bw_gw1_umma"):
        return "tensor", 2.0 * B * (Hd + 1) * h, "FLOP"
    if name == "adam":
        total = Hd * h + h + n * h + n
        # read g, m, v, theta; write m, v, theta (28 B per live param) + the fp16 pair of [W2 | b2] (4 B)
        return "hbm", 28.0 * total + 4.0 * n * (h + 1), "B"
    if name == "maxcut_energy":
        W = (n + 31) // 32
        return "hbm", 4.0 * B * W + 8.0 * E + 12.0 * B, "B"
    if name == "head_sample":
        return "latency", 2.0 * B * Hd * (h + Hd), "FLOP"
    return None, None, None


def run_ours(args):
    world, rank, local = dist_env()
    D = Dist(world, rank)
    import torch
    torch.cuda.set_device(local)
    from paper_2106_13308_b200 import _capi as K
    from paper_2106_13308_b200 import api

    g, gdesc = make_instance(args)
    n = args.n
    h = api.default_made_hidden(n)
    model = api.made_init(n, h, args.seed)
    Hd = int(model.degrees.max())
    B = args.minibatch
    hd = C.c_void_p()
    e = np.ascontiguousarray(g.edges, np.int32)
    K.check(K.lib.vqmc_gpu_create(local, n, h, K.ptr(model.degrees), K.ptr(model.parameters()), K.ptr(e), len(e),
                                  B, C.byref(hd)))
    if world > 1 or os.environ.get("VQMC_NCCL_SELF") == "1":  # (1 rank: exercises the overlapped path)
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            K.check(K.lib.vqmc_gpu_comm_unique_id(uid))
        b = D.bcast_bytes(bytes(uid))
        uid = (C.c_uint8 * 128).from_buffer_copy(b)
        K.check(K.lib.vqmc_gpu_comm_init(hd, uid, world, rank))
    K.check(K.lib.vqmc_gpu_adam_reset(hd))
    lr, b1, b2, eps = 0.01, 0.9, 0.999, 1e-8
    from paper_2106_13308_b200 import dp
    stream0 = dp.RankPlan(rank, world, 1).stream0  # worker w = rank -> stream (seed, w + 1)
    step = [0]

    def one_step(stats=None):
        step[0] += 1
        K.check(K.lib.vqmc_gpu_train_step(hd, B, 1, None, args.seed, stream0, step[0], lr, b1, b2, eps, step[0],
                                          stats))

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    for _ in range(max(args.warmup, 0)):
        one_step()
    # ---- timed region: the production path (CUDA-graph replay), whole-step CUDA events on the
    # library's stream, L2 flushed between steps outside the events ----
    K.check(K.lib.vqmc_gpu_set_phase_timing(hd, 1))
    one_step()  # (re)capture for the timing configuration
    one_step()
    K.check(K.lib.vqmc_gpu_synchronize(hd))
    clocks = ClockSampler()
    if rank == 0 and not args.profile:
        clocks.start()
    D.barrier()
    torch.cuda.synchronize()
    total_ms = 0.0
    pms = (C.c_float * 5)()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush (256 MB > 126 MB L2) between timed iterations, outside the events
        torch.cuda.synchronize()
        one_step()
        K.check(K.lib.vqmc_gpu_phase_times(hd, pms))
        total_ms += float(pms[0])
    K.check(K.lib.vqmc_gpu_synchronize(hd))
    torch.cuda.synchronize()
    D.barrier()
    clk = clocks.stop() if (rank == 0 and not args.profile) else None
    T = D.max(total_ms)
    ms_per_step = T / args.steps
    value = world * B * 1000.0 / ms_per_step

    # ---- kernel breakdown (roofline): per-kernel CUDA events recorded inside the replayed graph ----
    K.check(K.lib.vqmc_gpu_set_phase_timing(hd, 2))
    K.check(K.lib.vqmc_gpu_set_kernel_timing(hd, 1))
    one_step()
    one_step()
    ktimes: dict = {}
    kcount: dict = {}
    phase = np.zeros(5)
    names = C.create_string_buffer(32 * 128)
    kms = (C.c_float * 128)()
    cnt = C.c_int()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        one_step()
        K.check(K.lib.vqmc_gpu_phase_times(hd, pms))
        phase += np.array(list(pms))
        K.check(K.lib.vqmc_gpu_kernel_times(hd, names, kms, 128, C.byref(cnt)))
        for i in range(cnt.value):
            nm = names.raw[32 * i: 32 * i + 32].split(b"\0")[0].decode()
            ktimes[nm] = ktimes.get(nm, 0.0) + kms[i]
            kcount[nm] = kcount.get(nm, 0) + 1
    K.check(K.lib.vqmc_gpu_synchronize(hd))
    launches = int(round(sum(kcount.values()) / args.steps)) * args.steps

    # ---- timeline of the production (concurrent) schedule: start / end events of every kernel on
    # its own stream, relative to the step-start event (mean over K steps) ----
    K.check(K.lib.vqmc_gpu_set_phase_timing(hd, 1))
    K.check(K.lib.vqmc_gpu_set_kernel_timing(hd, 2))
    one_step()
    one_step()
    tl: dict = {}
    ks_, ke_ = (C.c_float * 128)(), (C.c_float * 128)()
    tl_total = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        one_step()
        K.check(K.lib.vqmc_gpu_phase_times(hd, pms))
        tl_total += pms[0]
        K.check(K.lib.vqmc_gpu_kernel_timeline(hd, names, ks_, ke_, 128, C.byref(cnt)))
        for i in range(cnt.value):
            nm = names.raw[32 * i: 32 * i + 32].split(b"\0")[0].decode()
            a = tl.setdefault(f"{i:02d} {nm}", [0.0, 0.0])
            a[0] += ks_[i]
            a[1] += ke_[i]
    K.check(K.lib.vqmc_gpu_synchronize(hd))
    # gW2 and dg1 on their SM partitions (vqmc_gpu_create: gW2 gets 80 SMs from N = 8192 up, else 64)
    gw2_sms = int(os.environ.get("VQMC_GW2_SMS", 80 if n >= 8192 else 64))
    conc = {}
    for nm, sms in (("bw_gw2_umma", gw2_sms), ("bw_dg1_umma", 148 - gw2_sms)):
        spans = [v for k, v in tl.items() if k[3:] == nm]
        if not spans:
            continue
        dur_ms = (spans[0][1] - spans[0][0]) / args.steps
        w_ = kernel_work(nm, n, h, Hd, B, len(e))[1]
        ach = w_ / (dur_ms * 1e-3) / 1e12
        pk = (measured_peaks() or {}).get("bf16_tflops_sustained", 1400.0)
        conc[nm] = {"timeline_us": round(1e3 * dur_ms, 2), "sms": sms, "achieved": ach, "unit": "TFLOP/s",
                    "frac_of_partition": ach / (pk * sms / 148.0)}
    timeline = {"step_ms": round(tl_total / args.steps, 5),
                "kernels": [{"kernel": k[3:], "start_us": round(1e3 * v[0] / args.steps, 2),
                             "end_us": round(1e3 * v[1] / args.steps, 2)} for k, v in sorted(tl.items())],
                "note": "production schedule (gW2 + Adam[W2|b2] on the side stream beside dg1 -> dz1 -> gW1 -> "
                        "Adam[W1|b1]); start = when the kernel's stream reached it (after its predecessors "
                        "and cross-stream waits), end = its completion; event nodes between kernels cost "
                        "~1-2 us each, so step_ms here exceeds ms_per_step"}

    # e2e: the public API call (blocking; per-step statistics copied to the host)
    K.check(K.lib.vqmc_gpu_set_phase_timing(hd, 0))
    K.check(K.lib.vqmc_gpu_set_kernel_timing(hd, 0))
    e2e = None
    if not args.profile:
        st = K.StepStats()
        for _ in range(2):  # untimed: the timing modes changed, so the step graph is re-captured
            one_step(C.byref(st))
        D.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one_step(C.byref(st))
        e2e_s = D.max(time.perf_counter() - t0)
        e2e = {"value": world * B * args.steps / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": C.sizeof(K.StepStats),
               "steps_per_s": args.steps / e2e_s,
               "note": "vqmc_gpu_train_step with stats_out (blocking, per-step stats D2H); the step's only "
                       "inputs are scalars (seed, stream, counter) - samples are generated on the device by "
                       "design (Philox), so there is no per-step H2D payload"}

    # final cut (evaluate, trainer.cpp:91-108) on the eval stream
    ev = np.empty(4)
    K.check(K.lib.vqmc_gpu_evaluate(hd, 1024, None, args.seed, api.kEvalStream, 0, K.ptr(ev)))

    if rank != 0:
        K.lib.vqmc_gpu_destroy(hd)
        return None

    # dominant kernel + roofline
    peaks = measured_peaks()
    avg = {k: ktimes[k] / kcount[k] for k in ktimes}
    share = {k: ktimes[k] / max(1e-9, sum(ktimes.values())) for k in ktimes}
    # the roofline object describes the largest kernel with a tensor or HBM bound that has the whole
    # GPU in the production schedule: the tail sampler GEMM (gW2 and dg1 run concurrently on two SM
    # partitions -- reported under "concurrent_gemms" from the timeline; their serial-pass times
    # describe a schedule that is not run, dg1's split count being planned for its partition).  The
    # head sampler, a serial dependency chain, is reported beside it under "head_latency".
    modelled = [k for k in ktimes if kernel_work(k, n, h, Hd, B, len(e))[0] in ("tensor", "hbm")]
    alone = [k for k in modelled if k not in ("bw_gw2_umma", "bw_dg1_umma", "adam")]
    dom = max(alone or modelled, key=lambda k: ktimes[k])
    bound, work, wunit = kernel_work(dom, n, h, Hd, B, len(e))
    traffic = None  # dram bytes per launch of that kernel from the committed ncu --set full capture
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom)
        except (OSError, ValueError):
            traffic = None
    roof = None
    if bound == "tensor":
        ach = work / (avg[dom] * 1e-3) / 1e12
        pk = peaks["bf16_tflops_sustained"] if peaks else 1400.0
        roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk,
                "traffic": traffic, "peak_src": "MEASURED_PEAKS.json bf16_tflops_sustained" if peaks else "fallback",
                "algorithmic_per_launch": work, "launch_ms": avg[dom],
                "note": "achieved = algorithmic (useful, single-pass) FLOPs / launch time.  Every operand is an "
                        "fp16 pair and the kernel issues 3 tcgen05 kind::f16 MMA passes (hi.hi + hi.lo + lo.hi, "
                        "fp32-grade), so its tensor-pipe ceiling for useful FLOPs is peak / 3; traffic = "
                        "dram read+write bytes per launch from profiles/traffic.json (ncu --set full)"}
    else:
        ach = work / (avg[dom] * 1e-3) / 1e9
        pk = peaks["hbm_gbs"] if peaks else 6650.0
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": pk, "unit": "GB/s", "frac": ach / pk,
                "traffic": traffic, "algorithmic_per_launch": work, "launch_ms": avg[dom]}
    # all tensor/hbm kernels for context
    kernels = {}
    for k in sorted(ktimes, key=lambda k: -ktimes[k]):
        b_, w_, u_ = kernel_work(k, n, h, Hd, B, len(e))
        ent = {"avg_ms": round(avg[k], 5), "share": round(share[k], 4)}
        if w_:
            ent["achieved"] = w_ / (avg[k] * 1e-3) / (1e12 if u_ == "FLOP" else 1e9)
            ent["unit"] = "TFLOP/s" if u_ == "FLOP" else "GB/s"
        kernels[k] = ent
    head_lat = None
    if "head_sample" in avg:  # the head's serial chain: cycles per sampled bit at the measured clock
        hz = (clk or {}).get("sm_mhz") or 1965.0
        head_lat = {"kernel": "head_sample", "launch_ms": avg["head_sample"], "bits": Hd,
                    "cycles_per_bit": avg["head_sample"] * 1e-3 * hz * 1e6 / max(Hd, 1),
                    "fp32_tflops": kernel_work("head_sample", n, h, Hd, B, len(e))[1] / (avg["head_sample"] * 1e-3) / 1e12,
                    "note": "latency-bound dependency chain over the first Hd bits; reported beside the roofline"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline and not args.profile:
        cpu = cpu_baseline(args, g, B)

    # SGD + SR step (the reference cannot form S at this size: B x d fp64 = 70 GB)
    sr = None
    if world == 1 and not args.profile and not args.no_sr:
        st = K.StepStats()
        cg_it, cg_res = C.c_int(0), C.c_double(0.0)
        iters = []

        def sr_step(i):
            K.check(K.lib.vqmc_gpu_train_step_sr(hd, B, 1, None, args.seed, stream0, 10_000 + i, 0.1, 1e-3, 1e-6, 200,
                                                 1, 1, C.byref(st), C.byref(cg_it), C.byref(cg_res)))
            iters.append(cg_it.value)

        sr_step(0)  # (first use allocates the CG buffers)
        K.check(K.lib.vqmc_gpu_synchronize(hd))
        iters.clear()
        t0 = time.perf_counter()
        for i in range(3):
            sr_step(1 + i)
        K.check(K.lib.vqmc_gpu_synchronize(hd))
        sr_ms = (time.perf_counter() - t0) * 1e3 / 3
        sr = {"ms_per_step": sr_ms, "samples_per_s": B * 1000.0 / sr_ms, "cg_iterations": iters,
              "ms_per_cg_iteration": sr_ms / max(1.0, float(np.mean(iters))),
              "workload": "SGD + SR (lambda 1e-3, tol 1e-6, centred), same instance and batch; CG on the "
                          "structured Fisher operator (the scores are never formed)",
              "timing": "host wall clock around 3 blocking vqmc_gpu_train_step_sr calls (the CG loop reads one "
                        "scalar per iteration)"}

    K.lib.vqmc_gpu_destroy(hd)
    line = {
        "metric": "samples/sec (VQMC training step, N=10k Max-Cut MADE)",
        "value": value,
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "steps_per_s": 1000.0 / ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 (fp64 accumulation for log-probs and energies; integer cuts)",
        "data": "synthetic (random 3-regular graph, random-init MADE; Philox uniforms)",
        "config": {"workload": f"Max-Cut N={n} ({gdesc}), MADE h={h}, AUTO sampler, ADAM lr=0.01",
                   "samples_per_gpu": B, "global_batch": world * B, "parallelism": f"dp{world}",
                   "l2": "flushed between timed iterations (256 MB write, outside the events)"},
        "phase_ms": {k: round(v / args.steps, 5) for k, v in
                     zip(["sample", "energy+weights", "backward", "allreduce", "adam+refresh"], phase)},
        "phase_ms_note": "phase and kernel events come from a second K-step pass (event nodes between kernels "
                         "add overhead); per-kernel events run the backward in the SERIAL schedule (one stream; "
                         "the timed steps overlap gW2 + its all-reduce with dg1 -> dz1 -> gW1 on a side stream); "
                         "ms_per_step uses whole-step events of the concurrent schedule only",
        "kernels": kernels,
        "timeline": timeline,
        "concurrent_gemms": conc,
        "head_latency": head_lat,
        "roofline": roof,
        "final_cut": {"best_cut": ev[2], "mean_cut": ev[3], "energy": ev[0], "note": "eval batch 1024 after "
                      f"{args.warmup + 2 * args.steps} training steps"},
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
        "graph": "each step is one captured CUDA graph replayed per iteration (vqmc_gpu_set_graph)",
        "cpu_baseline": cpu,
        "sr": sr,
    }
    return line


def cpu_baseline(args, g, B, steps=1, budget_s=None):
    """The reference algorithm (oracle restatement, fp64, n full forward passes per sampling
    call) on the host cores: workers = cores, minibatch B / cores each (effective batch B)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    cores = os.cpu_count() or 1
    workers = max(1, min(cores, B // 2))
    mbs = max(2, B // workers)
    budget = budget_s or args.cpu_seconds
    # calibrate: one bit
    cal = O.time_reference_step(args.n, g.edges, workers, mbs, seed=args.seed, bits_limit=1)
    per_bit = cal["sample_s"] / args.n
    bits = int(max(1, min(args.n, budget / max(per_bit, 1e-9))))
    runs = [O.time_reference_step(args.n, g.edges, workers, mbs, seed=args.seed, bits_limit=bits)
            for _ in range(steps)]
    step_s = float(np.mean([r["step_s"] for r in runs]))
    return {"value": workers * mbs / step_s, "unit": "samples/s", "cores": workers, "kind": "port",
            "steps_per_s": 1.0 / step_s, "extrapolated": bits < args.n, "bits_timed": bits,
            "cpu_model": cpu_model(), "nproc": cores,
            "sample": f"one reference iteration, {workers} worker threads x minibatch {mbs} (batch {workers * mbs}); "
                      f"sampler timed for the first {bits} of {args.n} bits (each bit is one full two-GEMM forward "
                      f"pass, sampler.cpp:47-48) and extrapolated x{args.n / bits:.1f}; energy, gradient, tree "
                      f"all-reduce and Adam timed in full; fp64 OpenBLAS dgemm, 1 thread per worker",
            "step_s": step_s, "sampler_s": runs[0]["sample_s"], "estimate_s": runs[0]["estimate_s"],
            "update_s": runs[0]["update_s"], "oracle": "oracle/vqmc_oracle.cpp (restated reference; Eigen absent)"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_instance(args):
    """The same synthetic instance as make_instance, generated by the oracle (the reference arm
    must not load the repo's own library)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    if args.graph == "regular3":
        e = O.random_regular_graph(args.n, 3, args.seed)
        return e, f"random 3-regular, |E|={len(e)}"
    e = O.random_maxcut_graph(args.n, args.seed)
    return e, f"reference G(n,3/4), |E|={len(e)}"


def validate_extrapolation(O, workers, mbs, seed, n=1000, bits=40):
    """One FULL reference iteration (all n sampler bits timed) against the per-bit extrapolation
    used at N = 10k (sampler timed for `bits` bits, x n / bits; every bit is one identical full
    two-GEMM forward pass, sampler.cpp:47-48; trainer.cpp:254 times the whole iteration)."""
    e = O.random_regular_graph(n, 3, seed)
    O.time_reference_step(n, e, workers, mbs, seed=seed, bits_limit=4)  # (warm the BLAS / threads)
    t0 = time.perf_counter()
    full = O.time_reference_step(n, e, workers, mbs, seed=seed, bits_limit=n)
    wall = time.perf_counter() - t0
    ext = O.time_reference_step(n, e, workers, mbs, seed=seed, bits_limit=bits)
    return {"n": n, "graph": "random 3-regular", "measured_step_s": full["step_s"], "measured_wall_s": wall,
            "extrapolated_step_s": ext["step_s"], "bits_timed_in_extrapolation": bits,
            "measured_over_extrapolated": full["step_s"] / ext["step_s"]}


def run_reference(args):
    """The reference algorithm (the oracle's restatement of proj/src/{sampler,models,trainer}.cpp,
    fp64, n full forward passes per sampling call; Eigen is absent so the reference itself cannot be
    built) on all host cores.  Imports only oracle/ (never the repo's package or its .so)."""
    world, rank, local = dist_env()
    if rank != 0:
        return None
    e, gdesc = oracle_instance(args)
    B = args.minibatch
    K_, W_ = max(1, args.steps), max(0, args.warmup)
    budget = max(2.0, min(20.0, 150.0 / (K_ + W_)))
    import pyoracle as O
    cores = os.cpu_count() or 1
    workers = max(1, min(cores, B // 2))
    mbs = max(2, B // workers)
    t_start = time.perf_counter()
    cal = O.time_reference_step(args.n, e, workers, mbs, seed=args.seed, bits_limit=1)
    per_bit = cal["sample_s"] / args.n
    bits = int(max(1, min(args.n, budget / max(per_bit, 1e-9))))
    for _ in range(W_):
        O.time_reference_step(args.n, e, workers, mbs, seed=args.seed, bits_limit=max(1, bits // 4))
    t_timed = time.perf_counter()
    runs = [O.time_reference_step(args.n, e, workers, mbs, seed=args.seed, bits_limit=bits) for _ in range(K_)]
    timed_wall = time.perf_counter() - t_timed
    step_s = float(np.mean([r["step_s"] for r in runs]))
    value = workers * mbs / step_s
    val = validate_extrapolation(O, workers, mbs, args.seed) if args.n > 1000 else None
    h = O.default_made_hidden(args.n)
    extrap = bits < args.n
    sample = (f"{workers} worker threads x minibatch {mbs}; per step the reference sampler runs the first {bits} of "
              f"{args.n} bits (one full forward pass each)" + (" and is extrapolated x n/bits" if extrap else "") +
              "; energy/gradient/all-reduce/Adam timed in full")
    return {"impl": "reference", "metric": "samples/sec (VQMC training step, N=10k Max-Cut MADE)", "value": value,
            "unit": "samples/s", "n_gpus": 0, "steps": K_, "warmup": W_, "ms_per_step": step_s * 1000.0,
            "steps_per_s": 1.0 / step_s, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"Max-Cut N={args.n} ({gdesc}), MADE h={h}, AUTO sampler, ADAM lr=0.01",
                       "samples_per_step": workers * mbs, "parallelism": f"{workers} host threads"},
            "extrapolated": extrap, "bits_timed": bits, "bits_total": args.n,
            "timed_region_wall_s": timed_wall, "run_wall_s": time.perf_counter() - t_start,
            "extrapolation_check": val, "nproc": cores, "cpu_model": cpu_model(),
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": workers, "kind": "port", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if args.impl == "reference":
        line = run_reference(args)
    else:
        line = run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
