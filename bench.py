#!/usr/bin/env python
"""bench.py — low-bit GeMM throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (default, BASELINE.json configs[4] = "c5"): TNN GeMM, A = 1,048,576 x
2048 ternary (P(0)=1/3), B = 2048 x 1024 ternary, int16 C; A rows sharded
contiguously over the N ranks, B replicated (weights: encoded + pack_b +
prepared once, untimed, as the reference bench does, bench.cpp:40-68).
Total work is fixed as N grows -> "scaling": "strong".  No collective on the
data path (north_star: NCCL only gathers outputs where a test requires it).

One step = one gemm_lowbit over this rank's rows with the encoded A planes
resident in HBM (the reference timing policy: encode and pack_b excluded,
bench.cpp:49,58).  L2 is flushed (256 MiB write + read) between steps, outside the
CUDA events that time each step's kernel.  value = 2*M*N*K / max-over-ranks of
the per-step device time, in TOPS.

e2e: the same metric through the reference-facing host call
(lowbit_gemm_lowbit_host: host A planes + host PackedB in, host int16 C out),
pinned host buffers, copies inside the timed region.

cpu_baseline / --impl reference: the reference library itself
(oracle/_ref/liblowbit_ref.so, built from /root/reference/proj/src with its
own flags) on a bounded row sample of the same workload, all host threads.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (mode, M, N, K, dist_a, dist_b, seed)   modes: 0 bnn, 1 tnn, 2 tbn
    "c1": (1, 360, 96, 256, 0, 0, 43),
    "c3": (0, 8192, 8192, 4096, 1, 1, 45),
    "c5": (1, 1048576, 1024, 2048, 0, 0, 47),
}
MODE_NAME = {0: "bnn", 1: "tnn", 2: "tbn"}
SWEEP = [(m, n, k) for m in (72, 120, 240, 360) for n in (24, 48, 72, 96) for k in (128, 256, 384, 512)]


def peaks():
    p = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
    except OSError:
        pass
    return {
        "hbm_gbs": p.get("hbm_gbs", 6650.0),
        "bf16_tflops": p.get("bf16_tflops", 1590.0),
        "bf16_tflops_sustained": p.get("bf16_tflops_sustained", 1400.0),
        "source": "measured (MEASURED_PEAKS.json)" if p else "fallback (B200_PROFILING.md)",
        "sm_max_mhz": p.get("sm_max_mhz", 1965.0),
    }


class ClockSampler:
    """Clocks + throttle reasons sampled during the timed region (NVML every
    5 ms; nvidia-smi -lms 100 as a fallback)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.stop = False
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nvml
        names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4}
        while not self.stop:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                act = ["Active" if r & bit else "Not Active" for bit in names.values()]
                self.lines.append(", ".join([str(sm), str(mx), "0"] + act))
            except Exception:
                pass
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml is not None:
            self.stop = True
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except OSError:
        return {}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref) on bounded samples — BASELINE.md §2
# ---------------------------------------------------------------------------
def _ref_lib(native=False):
    from oracle.oracle import REF_NATIVE_SO, REF_SO, Ref
    path = REF_NATIVE_SO if native else REF_SO
    return Ref(path) if Ref.available(path) else None


def cpu_gemm(ref, port, mode, M, N, K, da, db, seed, ids=(0, 1), threads=1, rows=None, target_s=None, reps=1,
             from_i8=False):
    """The reference gemm_lowbit (oracle/_ref, built from /root/reference/proj/src) on `rows` rows of a
    config, split over `threads` contiguous row shards (one std::thread each; the library is pure,
    kernels.cpp:23).  Policy of bench.cpp:214-233: one warm-up run, then the median of `reps` timed
    runs; encode(A) and pack_b excluded — unless from_i8, which times encode_* + gemm_lowbit ("from
    int8 A").  target_s: grow the row sample until one run takes ~target_s."""
    from oracle.oracle import a_mode_ternary, b_mode_ternary
    b = port.generate(db, seed, ids[1], K, N)
    b0, b1 = ref.encode(b, b_mode_ternary(mode))

    def run(r, reps_):
        r = min(r, M)
        a = port.generate(da, seed, ids[0], r, K)
        if from_i8:
            h = ref.bench_prepare_i8(mode, a, r, K, b0, b1, N, threads)
        else:
            a0, a1 = ref.encode(a, a_mode_ternary(mode))
            h = ref.bench_prepare(mode, a0, a1, r, K, b0, b1, N, threads)
        ref.bench_run(h)  # warm-up (bench.cpp:214)
        ts = []
        for _ in range(reps_):
            t0 = time.perf_counter()
            ref.bench_run(h)
            ts.append(time.perf_counter() - t0)
        ref.bench_free(h)
        return r, float(np.median(ts))

    if target_s is not None:
        # calibrate on whole 16-row tiles per shard (gemm_lowbit pads row blocks to 16, kernels.hpp:27);
        # thread start-up dominates tiny samples
        r, t = run(64 * threads, 1)
        while t < 0.2 * target_s and r < M:
            r, t = run(min(M, r * 4), 1)
        rows = int(min(M, max(r, target_s * r / t)))
    rows, t = run(rows or M, reps)
    return {"rows": rows, "seconds": t, "TOPS": 2.0 * rows * N * K / t / 1e12}


def reference_cpu_rate(cfg_name, target_s=8.0, threads=None, native=False, one_core_s=None):
    """Bounded-sample rate of the reference CPU path on config `cfg_name` at `threads` (default: all
    host threads), as a cpu_baseline object.  one_core_s: also a 1-thread figure on ~that many s."""
    from oracle.oracle import Port
    mode, M, N, K, da, db, seed = CONFIGS[cfg_name]
    ref = _ref_lib(native)
    if ref is None:
        return None
    port = Port()
    threads = threads or os.cpu_count() or 1
    r = cpu_gemm(ref, port, mode, M, N, K, da, db, seed, threads=threads, target_s=target_s)
    out = {"value": r["TOPS"], "unit": "TOPS", "cores": threads, "kind": "reference",
           "sample": f"{MODE_NAME[mode]} {r['rows']} x {N} x {K} rows of {cfg_name} (gemm_lowbit on {threads} "
                     f"row shards, encode/pack_b excluded, warm-up then timed), {r['seconds']:.2f} s",
           "seconds": r["seconds"], "build": "x86-64-v3" if native else "reference flags (-O3)"}
    if one_core_s:
        r1 = cpu_gemm(ref, port, mode, M, N, K, da, db, seed, threads=1, target_s=one_core_s)
        out["one_core"] = {"value": r1["TOPS"], "cores": 1, "sample": f"{r1['rows']} rows, {r1['seconds']:.2f} s"}
    return out


def cpu_baselines(threads=None):
    """BASELINE.md §2 beside every GPU number: the reference CPU path on this host for configs 1-5,
    on all host threads and on 1 core, its own -O3 build and the x86-64-v3 build, plus the
    "from int8 A" line (encode included).  Bounded samples; ~1 min in total."""
    from oracle.oracle import Port
    port = Port()
    threads = threads or os.cpu_count() or 1
    out = {}
    for native in (False, True):
        ref = _ref_lib(native)
        if ref is None:
            continue
        tag = "x86_64_v3" if native else "reference_build"
        # c1: the whole config, median of 5, 1 core (the reference bench's own policy)
        mode, M, N, K, da, db, seed = CONFIGS["c1"]
        r = cpu_gemm(ref, port, mode, M, N, K, da, db, seed, threads=1, reps=5)
        ri = cpu_gemm(ref, port, mode, M, N, K, da, db, seed, threads=1, reps=5, from_i8=True)
        out.setdefault("c1", {})[tag] = {
            "value": r["TOPS"], "unit": "TOPS", "cores": 1, "kind": "reference", "ms": r["seconds"] * 1e3,
            "from_int8": {"value": ri["TOPS"], "ms": ri["seconds"] * 1e3},
            "sample": "whole config, median of 5 after one warm-up (bench.cpp:214-233)"}
        # c2: the 64-shape TBN sweep, sum of the 64 medians, 1 core
        tot = tot_i8 = 0.0
        ops = 0.0
        for sidx, (m, n, k) in enumerate(SWEEP):
            r = cpu_gemm(ref, port, 2, m, n, k, 2, 1, 44, ids=(2 * sidx, 2 * sidx + 1), threads=1, reps=5)
            ri = cpu_gemm(ref, port, 2, m, n, k, 2, 1, 44, ids=(2 * sidx, 2 * sidx + 1), threads=1, reps=5,
                          from_i8=True)
            tot += r["seconds"]
            tot_i8 += ri["seconds"]
            ops += 2.0 * m * n * k
        out.setdefault("c2", {})[tag] = {
            "value": ops / tot / 1e12, "unit": "TOPS", "cores": 1, "kind": "reference", "ms_64_shapes": tot * 1e3,
            "from_int8": {"value": ops / tot_i8 / 1e12, "ms_64_shapes": tot_i8 * 1e3},
            "sample": "all 64 shapes, sum of medians of 5 (bench.cpp:196-234)"}
        # c3, c5: row samples on all threads and on 1 core
        for name, ts, t1 in (("c3", 3.0, 1.5), ("c5", 4.0, 1.5)):
            mode, M, N, K, da, db, seed = CONFIGS[name]
            r = cpu_gemm(ref, port, mode, M, N, K, da, db, seed, threads=threads, target_s=ts)
            r1 = cpu_gemm(ref, port, mode, M, N, K, da, db, seed, threads=1, target_s=t1)
            ri = cpu_gemm(ref, port, mode, M, N, K, da, db, seed, threads=threads, rows=r["rows"], from_i8=True)
            out.setdefault(name, {})[tag] = {
                "value": r["TOPS"], "unit": "TOPS", "cores": threads, "kind": "reference",
                "sample": f"{r['rows']} of {M} rows on {threads} row shards, {r['seconds']:.2f} s",
                "one_core": {"value": r1["TOPS"], "cores": 1, "sample": f"{r1['rows']} rows, {r1['seconds']:.2f} s"},
                "from_int8": {"value": ri["TOPS"], "cores": threads, "sample": f"{ri['rows']} rows"}}
        # c4: 64 single-image conv2d_lowbit calls (im2col + encode + pack_b + gemm, conv.cpp:33-59):
        # a sample of the batch's images, extrapolated to all 64
        ops4 = 2.0 * 200704 * 128 * 1152
        wt = port.generate(0, 46, 1, 9 * 128, 128)
        c4 = {}
        for thr, imgs in ((threads, min(64, 2 * threads)), (1, 2)):
            fm = port.generate(0, 46, 0, imgs * 56 * 56, 128).reshape(imgs, 56, 56, 128)
            ref.bench_conv(1, fm[:1], False, wt, False, 3, 3, 1, 1, 1)  # warm-up
            t0 = time.perf_counter()
            ref.bench_conv(1, fm, False, wt, False, 3, 3, 1, 1, thr)
            dt = time.perf_counter() - t0
            t64 = dt * 64.0 / imgs
            c4[thr] = {"value": ops4 / t64 / 1e12, "cores": thr, "ms_64_images": t64 * 1e3,
                       "sample": f"{imgs} of 64 images as single-image conv2d_lowbit calls on {thr} thread(s), "
                                 f"{dt:.2f} s"}
        out.setdefault("c4", {})[tag] = dict(c4[threads], unit="TOPS", kind="reference", one_core=c4[1])
    return out


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    mode, M, N, K, da, db, seed = CONFIGS[args.config]
    from oracle.oracle import Ref
    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/liblowbit_ref.so not built"}))
        return
    per_step = max(1.0, min(8.0, 60.0 / max(1, args.steps + args.warmup)))
    vals = []
    r = None
    for i in range(args.warmup + args.steps):
        r = reference_cpu_rate(args.config, target_s=per_step)
        if i >= args.warmup:
            vals.append(r["value"])
    v = float(np.mean(vals))
    ops = 2.0 * M * N * K
    line = {
        "impl": "reference", "metric": f"low-bit GeMM TOPS (MAC=2 ops), {MODE_NAME[mode]} {args.config}",
        "value": v, "unit": "TOPS", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ops / (v * 1e12) * 1e3,
        "ms_per_step_note": "extrapolated: the whole config's ops at the rate measured on a bounded row sample "
                            "(each step times one sample; rows are independent, gemm.cpp:35-51)",
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8 bit-planes / int16", "data": "synthetic (counter-based generator)",
        "config": {"workload": f"{args.config}: {MODE_NAME[mode]} M={M} N={N} K={K}, reference CPU path "
                               f"extrapolated from a bounded row sample per step"},
        "cpu_baseline": {"value": v, "unit": "TOPS", "cores": r["cores"], "kind": r["kind"], "sample": r["sample"]},
        "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto", choices=["auto", "tensor", "tensor_i8", "bitserial"])
    ap.add_argument("--layout", default="reference", choices=["nibbles", "lanes", "reference"],
                    help="A plane layout written by the (untimed) encode: reference (the reference's own bit "
                         "order, what the drop-in API exchanges) -> fp4 (kind::mxf4) K5 for large shapes, K3 for "
                         "launch-bound ones; nibbles -> K5; lanes -> int8 (kind::i8) K3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the per-config side measurements")
    ap.add_argument("--no-gather", action="store_true", help="N>1: skip the (untimed) NCCL gather of C to rank 0")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2205_09120_b200 as lb
    from paper_2205_09120_b200 import _lib as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # under torchrun (even at N = 1) the ranks form an NCCL group: barriers, the max-over-ranks
    # reduction and the output gather run exactly as at N = 8
    distributed = world > 1 or "LOCAL_RANK" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kernel = {"auto": lb.KERNEL_AUTO, "tensor": lb.KERNEL_TENSOR, "tensor_i8": lb.KERNEL_TENSOR_I8,
              "bitserial": lb.KERNEL_BITSERIAL}[args.kernel]

    mode, M, N, K, da, db, seed = CONFIGS[args.config]
    from paper_2205_09120_b200.shard import row_range
    r0, r1 = row_range(M, rank, world)
    m = r1 - r0

    # ---- untimed setup: inputs in HBM, weights prepared ----
    a = lb.generate(da, seed, 0, m, K, row0=r0)
    layout = {"reference": 0, "lanes": 1, "nibbles": 2}[args.layout] if args.kernel != "bitserial" else 0
    ap_ = lb.encode_binary(a, layout=layout) if mode == 0 else lb.encode_ternary(a, layout=layout)
    ap_ref = None
    if not args.no_e2e and layout != 0:  # the host drop-in exchanges reference-layout planes
        ap_ref = lb.encode_binary(a) if mode == 0 else lb.encode_ternary(a)
    del a
    b = lb.generate(db, seed, 1, K, N)
    bp = lb.encode_ternary(b) if mode == 1 else lb.encode_binary(b)
    pb = lb.pack_b(bp)
    w = lb.prepare_weights(pb)
    c = torch.empty((m, N), dtype=torch.int16, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    chosen = kernel if kernel else (lb.KERNEL_TENSOR if layout == 2 else lb.select_kernel(mode, m, N, K))

    def step():
        lb.gemm_lowbit(mode, ap_, w, (m, N, K), kernel=kernel, out=c)

    for _ in range(args.warmup):
        flush_l2(flush)
        step()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush_l2(flush)
            ev[i][0].record()
            step()
            ev[i][1].record()
        torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in ev]
    my_ms = float(np.sum(step_ms))
    t = torch.tensor([my_ms], dtype=torch.float64, device="cuda")
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    ops_total = 2.0 * M * N * K
    value = ops_total / (ms_per_step * 1e-3) / 1e12
    kernel_ms_avg = my_ms / args.steps
    ops_rank = 2.0 * m * N * K

    # ---- e2e through the reference-facing host call ----
    e2e = None
    if not args.no_e2e:
        sb = (K + 7) // 8
        h_a0 = torch.empty((m, sb), dtype=torch.uint8, pin_memory=True)
        src = ap_ref if ap_ref is not None else ap_
        h_a0.copy_(src.plane0[:, :sb])
        h_a1 = None
        if src.plane1 is not None:
            h_a1 = torch.empty((m, sb), dtype=torch.uint8, pin_memory=True)
            h_a1.copy_(src.plane1[:, :sb])
        del src
        h_pan = torch.empty(pb.panels.numel(), dtype=torch.uint8, pin_memory=True)
        h_pan.copy_(pb.panels)
        h_c = torch.empty((m, N), dtype=torch.int16, pin_memory=True)
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)

        def e2e_step():
            L.check(L.lib.lowbit_gemm_lowbit_host(
                mode, C.c_void_p(h_a0.data_ptr()), C.c_void_p(h_a1.data_ptr()) if h_a1 is not None else None,
                m, K, C.c_void_p(h_pan.data_ptr()), int(mode == 1), N, K, m, N, K, 4096,
                C.c_void_p(h_c.data_ptr()), kernel, stream), "e2e")

        e2e_steps = max(2, min(args.steps, 5))
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        es.record()
        for _ in range(e2e_steps):
            e2e_step()
        ee.record()
        torch.cuda.synchronize()
        te = torch.tensor([es.elapsed_time(ee) / e2e_steps], dtype=torch.float64, device="cuda")
        if distributed:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d = h_a0.numel() + (h_a1.numel() if h_a1 is not None else 0) + h_pan.numel()
        e2e = {"value": ops_total / (te.item() * 1e-3) / 1e12, "unit": "TOPS",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(h_c.numel() * 2),
               "ms_per_step": te.item(), "path": "lowbit_gemm_lowbit_host (pinned host planes + PackedB in, "
                                                 "int16 C out; includes B upload + prepare per call)"}
        # sanity: e2e output equals the device-resident output
        assert torch.equal(h_c.cuda(), c), "e2e output differs from device path"
        # the same call with PAGEABLE host buffers (numpy arrays, as most callers hold them): the
        # library stages them through pinned slots on a few host threads
        if world == 1:
            p_a0 = h_a0.numpy().copy()
            p_a1 = h_a1.numpy().copy() if h_a1 is not None else None
            p_pan = h_pan.numpy().copy()
            p_c = np.zeros((m, N), np.int16)  # pre-touched, like a reused output buffer

            def e2e_pageable():
                lb.gemm_lowbit_host(mode, p_a0, p_a1, m, K, p_pan, mode == 1, N, K, (m, N, K), kernel=kernel,
                                    out=p_c)
            e2e_pageable()
            ts = []
            for _ in range(e2e_steps):
                t0 = time.perf_counter()
                e2e_pageable()
                ts.append(time.perf_counter() - t0)
            assert np.array_equal(p_c, h_c.numpy()), "pageable e2e output differs"
            tp = float(np.mean(ts))
            e2e["pageable"] = {"value": ops_total / tp / 1e12, "unit": "TOPS", "ms_per_step": tp * 1e3,
                               "path": "lowbit_gemm_lowbit_host with pageable (numpy) host buffers, host clock "
                                       "around the synchronous call"}
            del p_a0, p_a1, p_pan, p_c
            e2e["cpp_dropin"] = cpp_dropin_e2e(mode, M, N, K, seed)
        del h_a0, h_a1, h_c
        ap_ref = None

    gather = None
    if distributed and not args.no_gather:
        # NCCL output gather to rank 0 (only where a consumer needs the whole C;
        # not part of `value`): int16 shards travel as bytes
        from paper_2205_09120_b200.shard import gather_rows
        dist.barrier()
        torch.cuda.synchronize()
        gs, ge = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gs.record()
        full = gather_rows(c, M)
        ge.record()
        torch.cuda.synchronize()
        tg = torch.tensor([gs.elapsed_time(ge)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        moved = (M - (r1 - r0)) * N * 2
        gather = {"ms": tg.item(), "bytes_into_rank0": moved, "GB/s": moved / (tg.item() * 1e-3) / 1e9,
                  "collective": "torch.distributed.gather (NCCL) of int16 shards as bytes"}
        del full
    pk = peaks()
    achieved = ops_rank / (kernel_ms_avg * 1e-3) / 1e12
    fp4 = chosen == lb.KERNEL_TENSOR and layout != 1  # K5 reads NIBBLES and REFERENCE planes, K3 LANES
    kkey = ("fp4" if fp4 else "tensor") if chosen in (lb.KERNEL_TENSOR, lb.KERNEL_TENSOR_I8) else "bitserial"
    traffic = load_traffic().get(f"{args.config}:{kkey}")
    if fp4:
        # dense fp4 tcgen05 = 4x bf16 per SM-clock (9 vs 2.25 PF spec), scaled from the measured bf16 burst
        tensor_peak = 4.0 * pk["bf16_tflops"]
        roof = {"bound": "tensor", "achieved": achieved, "peak": tensor_peak, "unit": "TOP/s",
                "frac": achieved / tensor_peak, "traffic": traffic,
                "kernel": "gemm_fp4_pair_kernel (tcgen05.mma.cta_group::2 kind::mxf4, unit block scales)",
                "peak_source": f"4 x bf16 dense {pk['bf16_tflops']} TFLOP/s (fp4 = 4x bf16 rate), {pk['source']}",
                # the fp4 pair MMA's own measured issue rate (tools/micro/mma_rate.cu, random operands,
                # profiles/r01/mma_microbench.txt): a stricter denominator than the bf16-derived peak
                "mma_issue_peak_measured": {"value": 8843.0, "frac": achieved / 8843.0,
                                            "source": "tools/micro/mma_rate.cu: 128 cycles per 256x256x64 "
                                                      "pair MMA at 1.82 GHz"},
                "algorithmic_ops_per_launch": ops_rank}
    elif chosen in (lb.KERNEL_TENSOR, lb.KERNEL_TENSOR_I8):
        tensor_peak = 2.0 * pk["bf16_tflops"]  # dense int8 tcgen05 = 2x bf16 per SM-clock (4.5 vs 2.25 PF spec)
        roof = {"bound": "tensor", "achieved": achieved, "peak": tensor_peak, "unit": "TOP/s",
                "frac": achieved / tensor_peak, "traffic": traffic,
                "kernel": "gemm_tc_pair_kernel (tcgen05.mma.cta_group::2 kind::i8)",
                "peak_source": f"2 x bf16 dense {pk['bf16_tflops']} TFLOP/s, {pk['source']}",
                "algorithmic_ops_per_launch": ops_rank}
    else:
        popc_peak = 148 * 16 * 32 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12 / (2 if mode == 1 else 1)
        roof = {"bound": "popc", "achieved": achieved, "peak": popc_peak, "unit": "TOP/s",
                "frac": achieved / popc_peak, "traffic": traffic, "kernel": "gemm_bitserial_kernel",
                "peak_source": "148 SMs x 16 POPC/clk x 32 bits x 2 ops x max clock (TNN: 2 POPC per word)"}

    cpu = None
    cpu_all = {}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu_all = cpu_baselines()
            cpu = dict(cpu_all[args.config]["reference_build"])
            if "x86_64_v3" in cpu_all[args.config]:
                cpu["x86_64_v3"] = cpu_all[args.config]["x86_64_v3"]
        except Exception as e:  # never let the baseline break the bench line
            cpu = {"value": None, "error": repr(e)}

    extra = {}
    if rank == 0 and world == 1 and not args.no_extra:
        extra = side_configs(lb, torch, flush, pk)
    for name, cb in cpu_all.items():  # the reference CPU path beside every GPU number
        extra.setdefault(name, {})["cpu_baseline"] = cb

    if rank == 0:
        line = {
            "metric": f"low-bit GeMM TOPS (MAC=2 ops), {MODE_NAME[mode]} {args.config}",
            "value": value, "unit": "TOPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": ("u8 bit-planes in, packed e2m1 (fp4) tensor-core MMA with unit block scales, f32 accumulate "
                      "(exact: |partial sums| <= 32767), int16 out" if fp4 else
                      "u8 bit-planes in, int8 tensor-core MMA, int32 accumulate, int16 out"
                      if chosen in (lb.KERNEL_TENSOR, lb.KERNEL_TENSOR_I8, lb.KERNEL_TENSOR_1CTA) else
                      "u8 bit-planes in, LOP3 + POPC, int32 accumulate, int16 out"),
            "data": "synthetic (counter-based splitmix64 generator, BASELINE.json distributions)",
            "config": {"workload": f"{args.config}: {MODE_NAME[mode]} GeMM M={M} N={N} K={K} int16 C, "
                                   f"A rows sharded over {world} GPU(s), B replicated",
                       "global_rows": M, "rows_per_rank": M // world, "l2": "flushed between steps (256 MiB write + read back, clean lines)",
                       "kernel": {1: "bitserial", 2: "tensor (fp4 K5)" if fp4 else "tensor (int8 K3)",
                                  4: "tensor (int8 K3)"}.get(chosen, str(chosen)),
                       "a_layout": {2: "nibbles (B200 nibble-interleaved bit planes from K1)",
                                    1: "lanes (B200 lane-interleaved bit planes from K1)",
                                    0: "reference (the reference's own plane encoding, core.hpp:3-10: what "
                                       "the drop-in API hands the library)"}[layout],
                       "parallelism": f"row-shard x{world}"},
            "gpu_launches": args.steps, "clocks": clk.summary(), "roofline": roof, "cpu_baseline": cpu,
            "e2e": e2e, "gather": gather, "per_config": extra,
        }
        print(json.dumps(line))
    if distributed:
        dist.destroy_process_group()


def cpp_dropin_e2e(mode, M, N, K, seed, iters=3):
    """End to end through the C++ drop-in exactly as a reference caller uses it: std::vector planes
    in, `Int16Matrix c = lowbit::gemm_lowbit(...)` out (cpp/bench/dropin_e2e.cpp; host clock around
    each call, result allocation included — the reference allocates it too, gemm.cpp:79-112)."""
    exe = os.path.join(ROOT, "paper_2205_09120_b200", "cpp", "build", "dropin_e2e")
    if not os.path.exists(exe):
        return {"unavailable": "cpp/build/dropin_e2e not built"}
    try:
        r = subprocess.run([exe, str(mode), str(M), str(N), str(K), str(iters), str(seed)], capture_output=True,
                           text=True, timeout=600)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode != 0 or not line:
            return {"error": f"rc={r.returncode} {r.stderr[-300:]}"}
        d = json.loads(line[-1])
        return {"value": d["TOPS"], "unit": "TOPS", "ms_per_step": d["ms_mean"],
                "h2d_bytes_per_step": d["h2d_bytes_per_call"], "d2h_bytes_per_step": d["d2h_bytes_per_call"],
                "equal_device_path": d["equal_device_path"],
                # the zero-initialised Int16Matrix the reference API returns by value, allocated alone,
                # and the call's rate without it (the library's own share of the call)
                "result_alloc_ms": d.get("result_alloc_ms_median"),
                "value_excluding_result_alloc": (2.0 * M * N * K / ((d["ms_mean"] - d["result_alloc_ms_median"]) * 1e-3)
                                                 / 1e12 if d.get("result_alloc_ms_median") is not None and
                                                 d["ms_mean"] > d["result_alloc_ms_median"] else None),
                "path": "C++ drop-in lowbit::gemm_lowbit(mode, TernaryPackedMatrix, PackedB, dims) -> Int16Matrix, "
                        "std::vector buffers, host clock, result allocation included"}
    except Exception as e:
        return {"error": repr(e)}


def cpp_dropin_conv(batch, h, w, c, cout, seed, iters=3):
    """Config 4 as `batch` single-image conv2d_lowbit calls through the C++ drop-in
    (cpp/bench/dropin_e2e.cpp conv)."""
    exe = os.path.join(ROOT, "paper_2205_09120_b200", "cpp", "build", "dropin_e2e")
    if not os.path.exists(exe):
        return {"unavailable": "cpp/build/dropin_e2e not built"}
    try:
        r = subprocess.run([exe, "conv", "1", str(batch), str(h), str(w), str(c), str(cout), str(iters), str(seed)],
                           capture_output=True, text=True, timeout=600)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode != 0 or not line:
            return {"error": f"rc={r.returncode} {r.stderr[-300:]}"}
        d = json.loads(line[-1])
        return {"ms_64_images": d["ms_median"], "TOPS": d["TOPS"], "equal_device_path": d["equal_device_path"],
                "path": "C++ drop-in: 64 x lowbit::conv2d_lowbit(tnn, FeatureMap, SignMatrix, ConvSpec) -> "
                        "IntFeatureMap, host clock (each call uploads its image, runs K7, widens to int32 and "
                        "downloads; the weights are encoded, packed, uploaded and prepared by the first call "
                        "and reused while they are unchanged)"}
    except Exception as e:
        return {"error": repr(e)}


def flush_l2(flush):
    """Evict L2 between timed steps: write a 256 MiB buffer (2x the 126 MB L2),
    then read it back so the lines left in L2 are clean — otherwise the next
    timed kernel pays for writing the flush buffer's dirty lines to HBM
    (~126 MB, ~19 us: half of a c4 conv)."""
    import torch
    flush.zero_()
    flush.view(torch.int64).sum()


def time_device(torch, fn, flush, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush_l2(flush)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def graph_time(torch, fn, reps=20, inner=1):
    """Device time of fn() captured `inner` times back to back in one CUDA graph,
    replayed `reps` times (removes the host/ctypes launch path from the
    measurement), per fn().  With inner = 1 a short fn() is bound by the host's
    graph-replay rate (~10 us per replay here), not by the GPU; inner > 1
    amortises that and gives the device time of fn() in a stream of calls."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(inner):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / inner


def graph_time_flushed_avg(torch, fn, flush, reps=10):
    """Device time of fn() with a cold L2, averaged over `reps`: one CUDA graph
    of reps x (L2 flush, fn) minus one of reps x (L2 flush), each replayed and
    timed with events.  (A single short kernel timed alone is quantised by the
    event clock: ~2 us steps on this pool.)"""
    fn()
    flush_l2(flush)
    torch.cuda.synchronize()

    def timed(with_fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                flush_l2(flush)
                if with_fn:
                    fn()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            g.replay()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return float(np.median(ts))

    return (timed(True) - timed(False)) / reps


def side_configs(lb, torch, flush, pk):
    """BASELINE.json configs 1-4 at N=1: device time per kernel, TOPS and the
    fraction of the binding roofline.  Small configs (c1, c2) are timed as
    CUDA-graph replays (launch-latency bound); c3/c4 with events + L2 flush."""
    import ctypes as C
    L = lb._lib
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    out = {}
    tensor_peak = 2.0 * pk["bf16_tflops"]
    popc = lambda mode: 148 * 16 * 32 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12 / (2 if mode == 1 else 1)
    kernels = (("tensor", lb.KERNEL_TENSOR), ("bitserial", lb.KERNEL_BITSERIAL))
    fp4_peak = 4.0 * pk["bf16_tflops"]
    # (name, A plane layout, kernel id, peak): K5 fp4 from the reference encoding (what AUTO runs) and
    # from nibble-interleaved planes, K3 int8 from lane-interleaved planes, K2 bit-serial
    variants = (("tensor_fp4", 0, lb.KERNEL_TENSOR, "fp4"), ("tensor_fp4_nibbles", 2, lb.KERNEL_TENSOR, "fp4"),
                ("tensor_i8_lanes", 1, lb.KERNEL_TENSOR, "i8"), ("bitserial", 0, lb.KERNEL_BITSERIAL, "popc"),
                ("auto_reference_planes", 0, lb.KERNEL_AUTO, "auto"))
    for name in ("c1", "c3"):
        mode, M, N, K, da, db, seed = CONFIGS[name]
        a = lb.generate(da, seed, 0, M, K)
        planes = {lay: (lb.encode_binary(a, layout=lay) if mode == 0 else lb.encode_ternary(a, layout=lay))
                  for lay in (0, 1, 2)}
        b = lb.generate(db, seed, 1, K, N)
        w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(b) if mode == 1 else lb.encode_binary(b)))
        c = torch.empty((M, N), dtype=torch.int16, device="cuda")
        res = {}
        for kn, lay, kid, pkind in variants:
            f = lambda: lb.gemm_lowbit(mode, planes[lay], w, (M, N, K), kernel=kid, out=c)
            ms = graph_time(torch, f, reps=10, inner=20) if name == "c1" else time_device(torch, f, flush)
            tops = 2.0 * M * N * K / (ms * 1e-3) / 1e12
            if pkind == "auto":  # the kernel lowbit_select_kernel picks for this shape
                pkind = "fp4" if lb.select_kernel(mode, M, N, K) == lb.KERNEL_TENSOR else "i8"
            peak = {"fp4": fp4_peak, "i8": tensor_peak}.get(pkind) or popc(mode)
            res[kn] = {"ms": ms, "TOPS": tops, "frac": tops / peak,
                       "bound": "popc" if kn == "bitserial" else "tensor"}
        res["auto"] = {2: "tensor_fp4", 3: "tensor_1cta (int8, single-CTA; reference planes)",
                       4: "tensor_i8 (reference planes)"}.get(lb.select_kernel(mode, M, N, K))
        # "from int8 A" (BASELINE.md §2 second line): the sign matrix in HBM, encode included
        pl = lb.empty_planes(M, K, mode != 0)

        def enc_gemm():
            L.check(L.lib.lowbit_encode_ex(int(mode != 0), 0, C.c_void_p(a.data_ptr()), M, K, K,
                                           C.c_void_p(pl.plane0.data_ptr()),
                                           C.c_void_p(pl.plane1.data_ptr()) if pl.plane1 is not None else None,
                                           pl.pitch, None, st), "encode")
            lb.gemm_lowbit(mode, pl, w, (M, N, K), out=c)
        for kn, f in (("from_int8_encode_then_auto", enc_gemm),
                      ("from_int8_gemm_i8", lambda: lb.gemm_lowbit_i8(mode, a, w, (M, N, K), out=c))):
            ms = graph_time(torch, f, reps=10, inner=20) if name == "c1" else time_device(torch, f, flush)
            res[kn] = {"ms": ms, "TOPS": 2.0 * M * N * K / (ms * 1e-3) / 1e12}
        if name == "c1":  # one call alone: a 1-call graph per replay (bound by the host's replay rate)
            res["auto_single_graph_replay_ms"] = graph_time(
                torch, lambda: lb.gemm_lowbit(mode, planes[0], w, (M, N, K), kernel=lb.KERNEL_AUTO, out=c))
        res["from_int8_encode_then_auto"]["path"] = "K1 encode (reference planes) + lowbit_gemm AUTO: two launches"
        res["from_int8_gemm_i8"]["path"] = "lowbit_gemm_i8: int8 A by TMA straight into tcgen05 kind::i8"
        res["timing"] = ("device time per call in a CUDA graph of 20 back-to-back calls (launch gaps included)"
                         if name == "c1" else "events, L2 flushed")
        out[name] = res
    # c2: the 64-shape TBN sweep (one launch per shape), captured as one graph
    aps, ws, cs = [], [], []
    for s, (M, N, K) in enumerate(SWEEP):
        a = lb.generate(2, 44, 2 * s, M, K)
        b = lb.generate(1, 44, 2 * s + 1, K, N)
        aps.append(lb.encode_ternary(a))
        ws.append(lb.prepare_weights(lb.pack_b(lb.encode_binary(b))))
        cs.append(torch.empty((M, N), dtype=torch.int16, device="cuda"))
    ops = sum(2.0 * M * N * K for M, N, K in SWEEP)
    res = {}
    for kn, kid in (("auto", lb.KERNEL_AUTO),) + kernels:
        def sweep():
            for s, (M, N, K) in enumerate(SWEEP):
                lb.gemm_lowbit(2, aps[s], ws[s], (M, N, K), kernel=kid, out=cs[s])
        ms = graph_time(torch, sweep, reps=10, inner=4)
        res[kn] = {"ms_64_shapes": ms, "us_per_shape": ms * 1e3 / 64, "TOPS": ops / (ms * 1e-3) / 1e12}
    probs = [(aps[s], ws[s], cs[s]) for s in range(len(SWEEP))]
    ms = graph_time(torch, lambda: lb.gemm_grouped(2, probs), reps=10, inner=20)
    ms1 = graph_time(torch, lambda: lb.gemm_grouped(2, probs), reps=20)
    res["grouped_one_launch"] = {"ms_64_shapes": ms, "us_per_shape": ms * 1e3 / 64, "TOPS": ops / (ms * 1e-3) / 1e12,
                                 "ms_single_graph_replay": ms1}
    # from int8 A: the 64 encodes (one launch each) + the grouped GeMM launch, one graph
    a8 = [lb.generate(2, 44, 2 * s, M, K) for s, (M, N, K) in enumerate(SWEEP)]

    def sweep_i8():
        for s, (M, N, K) in enumerate(SWEEP):
            L.check(L.lib.lowbit_encode_ex(1, 0, C.c_void_p(a8[s].data_ptr()), M, K, K,
                                           C.c_void_p(aps[s].plane0.data_ptr()), C.c_void_p(aps[s].plane1.data_ptr()),
                                           aps[s].pitch, None, st), "encode")
        lb.gemm_grouped(2, probs)
    ms = graph_time(torch, sweep_i8, reps=10, inner=10)
    res["from_int8_grouped"] = {"ms_64_shapes": ms, "us_per_shape": ms * 1e3 / 64, "TOPS": ops / (ms * 1e-3) / 1e12,
                                "path": "64 K1 encodes + one grouped bit-serial launch, one graph"}
    res["timing"] = ("device time per sweep: a CUDA graph of several back-to-back sweeps (64 launches, or 1 grouped "
                     "launch), replayed; ms_single_graph_replay: one sweep per graph replay (host replay-rate bound)")
    out["c2"] = res
    # c4: conv 64x56x56x128, 3x3 -> 128, s1 p1 (K4 fused im2col+encode + GeMM)
    fm = lb.generate(0, 46, 0, 64 * 56 * 56, 128).view(64, 56, 56, 128)
    wt = lb.generate(0, 46, 1, 9 * 128, 128)
    w = lb.prepare_weights(lb.pack_b(lb.encode_ternary(wt)))
    ws_bytes = int(lb._lib.lib.lowbit_conv2d_workspace_bytes(1, 64, 56, 56, 128, 3, 3, 1, 1))
    wsp = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    o = torch.empty((64, 56, 56, 128), dtype=torch.int16, device="cuda")
    ops4 = 2.0 * 200704 * 128 * 1152
    res = {}
    conv_paths = (("tensor_fp4", lb.KERNEL_TENSOR, fp4_peak,
                   "K7T: fused halo conv (int8 halo by TMA, e2m1 packed in smem, taps as UMMA row offsets, "
                   "filter resident in tensor memory, kind::mxf4, bias MMA + pack::16b epilogue), one launch"),
                  ("tensor_i8", lb.KERNEL_TENSOR_I8, tensor_peak,
                   "int8 implicit GeMM: im2col TMA over the int8 map -> tcgen05 kind::i8"),
                  ("bitserial", lb.KERNEL_BITSERIAL, popc(1), "K4 fused im2col+encode -> K2 bit-serial"))
    for kn, kid, peak, path in conv_paths:
        ms = graph_time_flushed_avg(torch, lambda: lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=kid, out=o,
                                                                    workspace=wsp), flush)
        res[kn] = {"ms": ms, "TOPS": ops4 / (ms * 1e-3) / 1e12, "frac": ops4 / (ms * 1e-3) / 1e12 / peak,
                   "path": path}
        if kn == "tensor_fp4":  # the conv's true bound: HBM (int8 map in, int16 map out, once each)
            c4_bytes = 64 * 56 * 56 * 128 + 64 * 56 * 56 * 128 * 2
            res[kn]["frac_hbm"] = c4_bytes / (ms * 1e-3) / 1e9 / pk["hbm_gbs"]
            res[kn]["algorithmic_bytes"] = c4_bytes
            ms10 = graph_time(torch, lambda: lb.conv2d_lowbit(1, fm, False, w, 3, 3, 1, 1, kernel=kid, out=o,
                                                              workspace=wsp), reps=10, inner=10)
            res[kn]["ms_back_to_back"] = ms10
    res["auto"] = "tensor_fp4"
    res["timing"] = ("cuda graph of 10 x (L2 flush, conv) minus one of 10 x (L2 flush), averaged (single short "
                     "launches are quantised by the event clock); ms_back_to_back: per conv in a graph of 10 back-to-back convs, "
                     "warm L2")
    # K4 alone (HBM-bound): int8 NHWC in, two bit planes out
    pitch = lb.plane_pitch(1152)
    p0 = wsp[: 200704 * pitch]
    p1 = wsp[200704 * pitch: 2 * 200704 * pitch]
    k4 = lambda: L.check(L.lib.lowbit_conv_encode(0, C.c_void_p(fm.data_ptr()), 64, 56, 56, 128, 3, 3, 1, 1, 0,
                                                  C.c_void_p(p0.data_ptr()), C.c_void_p(p1.data_ptr()), pitch,
                                                  None, st))
    ms = time_device(torch, k4, flush)
    k4_bytes = 64 * 56 * 56 * 128 + 2 * 200704 * pitch
    res["k4_encode"] = {"ms": ms, "GB/s": k4_bytes / (ms * 1e-3) / 1e9,
                        "frac_hbm": k4_bytes / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], "algorithmic_bytes": k4_bytes}
    # config 4 through the C++ drop-in exactly as a reference caller runs the batch: 64 single-image
    # lowbit::conv2d_lowbit(mode, FeatureMap, SignMatrix, ConvSpec) calls (conv.hpp:64-65), host
    # clock, std::vector in / IntFeatureMap out (the reference packs the weights per call, conv.cpp:49; the
    # drop-in encodes, packs and prepares them on the first call and reuses them while they are unchanged)
    res["cpp_dropin"] = cpp_dropin_conv(64, 56, 56, 128, 128, 46)
    out["c4"] = res
    # c5 "from int8 A": the int8 sign matrix straight to the tensor cores (no encode)
    a = lb.generate(0, 47, 0, 1048576, 2048)
    w5 = lb.prepare_weights(lb.pack_b(lb.encode_ternary(lb.generate(0, 47, 1, 2048, 1024))))
    c5 = torch.empty((1048576, 1024), dtype=torch.int16, device="cuda")
    ms = time_device(torch, lambda: lb.gemm_lowbit_i8(1, a, w5, (1048576, 1024, 2048), out=c5), flush, reps=10)
    ops5 = 2.0 * 1048576 * 1024 * 2048
    out["c5_from_int8"] = {"ms": ms, "TOPS": ops5 / (ms * 1e-3) / 1e12, "frac": ops5 / (ms * 1e-3) / 1e12 / tensor_peak,
                           "path": "lowbit_gemm_i8: int8 A tiles by TMA (128B swizzle) -> tcgen05 kind::i8"}
    # the same product from the int8 sign matrix through K1 (nibble planes) + K5 (fp4): two launches
    planes = lb.empty_planes(1048576, 2048, True)
    planes.layout = 2

    def via_planes():
        L.check(L.lib.lowbit_encode_ex(1, 2, C.c_void_p(a.data_ptr()), 1048576, 2048, 2048,
                                       C.c_void_p(planes.plane0.data_ptr()), C.c_void_p(planes.plane1.data_ptr()),
                                       planes.pitch, None, st), "encode")
        lb.gemm_lowbit(1, planes, w5, (1048576, 1024, 2048), out=c5)
    ms = time_device(torch, via_planes, flush, reps=10)
    out["c5_from_int8_via_fp4"] = {"ms": ms, "TOPS": ops5 / (ms * 1e-3) / 1e12,
                                   "frac": ops5 / (ms * 1e-3) / 1e12 / fp4_peak,
                                   "path": "K1 encode (NIBBLES planes, HBM-bound) + K5 fp4 GeMM"}
    # K2 (bit-serial, LOP3 + POPC) on c5: north_star's primary kernel on the largest TNN shape
    p5 = lb.encode_ternary(a)
    ms = time_device(torch, lambda: lb.gemm_lowbit(1, p5, w5, (1048576, 1024, 2048), kernel=lb.KERNEL_BITSERIAL,
                                                   out=c5), flush, reps=3)
    out["c5_bitserial"] = {"ms": ms, "TOPS": ops5 / (ms * 1e-3) / 1e12, "frac": ops5 / (ms * 1e-3) / 1e12 / popc(1),
                           "bound": "popc", "path": "K2 gemm_bitserial_kernel on reference planes"}
    del p5
    p5 = lb.encode_ternary(a, layout=2)
    ms = time_device(torch, lambda: lb.gemm_lowbit(1, p5, w5, (1048576, 1024, 2048), out=c5), flush, reps=10)
    out["c5_fp4_nibbles"] = {"ms": ms, "TOPS": ops5 / (ms * 1e-3) / 1e12, "frac": ops5 / (ms * 1e-3) / 1e12 / fp4_peak,
                             "path": "K5 on NIBBLES planes (canonical fp4 B section)"}
    del p5, c5, w5
    # K1 encode of c5's A (HBM-bound): 2 GiB int8 in, 2 x 512 MiB planes out
    eb = 1048576 * 2048 + 2 * 1048576 * planes.pitch
    for lay, name in ((2, "k1_encode_c5_nibbles"), (1, "k1_encode_c5_lanes"), (0, "k1_encode_c5_reference_layout")):
        enc = lambda: L.check(L.lib.lowbit_encode_ex(1, lay, C.c_void_p(a.data_ptr()), 1048576, 2048, 2048,
                                                     C.c_void_p(planes.plane0.data_ptr()),
                                                     C.c_void_p(planes.plane1.data_ptr()), planes.pitch, None, st))
        ms = time_device(torch, enc, flush, reps=5)
        out[name] = {"ms": ms, "GB/s": eb / (ms * 1e-3) / 1e9, "frac_hbm": eb / (ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                     "algorithmic_bytes": eb}
    return out


if __name__ == "__main__":
    main()
