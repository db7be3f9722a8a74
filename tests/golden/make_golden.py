"""Generate the golden fixtures from the REFERENCE library itself.

    python tests/golden/make_golden.py [--big]

Runs in the build container only (needs oracle/_ref/liblowbit_ref.so, built
by `make -C oracle` from /root/reference/proj/src).  Inputs come from the
counter-based generator (oracle/lowbit_oracle.c orc_generate, identical to
the GPU's lowbit_generate), so every case is reproducible from (dist, seed,
matrix_id, shape) alone; the fixtures store reference OUTPUTS:

  golden_small.npz     encode planes, pack_b panels, gemm_lowbit outputs and
                       conv2d_lowbit outputs for small cases (full arrays)
  golden_configs.json  BASELINE.json configs 1-5: sha256 of the reference's
                       int16 C (row-major, little-endian) — c1 and c2 also
                       as full arrays in golden_small.npz; c3-c5 (--big) as
                       hashes only (128 MiB / 25.7 MB / 2 GiB outputs)
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import BNN, TNN, TBN, Port, Ref, a_mode_ternary, b_mode_ternary  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SMALL = os.path.join(HERE, "golden_small.npz")
CONFIGS = os.path.join(HERE, "golden_configs.json")

# dist ids of the generator
UNI3, PM1, SPARSE3 = 0, 1, 2

SWEEP_M = (72, 120, 240, 360)
SWEEP_N = (24, 48, 72, 96)
SWEEP_K = (128, 256, 384, 512)


def sweep_shapes():
    return [(m, n, k) for m in SWEEP_M for n in SWEEP_N for k in SWEEP_K]


def mode_dists(mode):
    return (PM1 if mode == BNN else UNI3), (UNI3 if mode == TNN else PM1)


def sha(c: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(c, dtype="<i2").tobytes()).hexdigest()


SMALL_GEMM = [(1, 1, 1), (15, 7, 9), (17, 9, 500), (70, 25, 7), (1, 25, 500), (72, 24, 128), (120, 96, 256),
              (33, 19, 700), (240, 48, 384), (129, 130, 333), (16, 8, 32767)]


def make_small(port: Port, ref: Ref) -> dict:
    out = {}
    # encode + pack_b
    for case, (rows, cols) in enumerate([(1, 8), (7, 13), (9, 17), (3, 64), (5, 100), (16, 504), (33, 129)]):
        for ternary in (0, 1):
            v = port.generate(UNI3 if ternary else PM1, 1000 + case, ternary, rows, cols)
            p0, p1 = ref.encode(v, bool(ternary))
            out[f"enc_{case}_{ternary}_p0"] = p0
            if ternary:
                out[f"enc_{case}_{ternary}_p1"] = p1
            pb = ref.pack_b(p0, p1, rows, cols)  # treat v as a K x N weight matrix
            out[f"packb_{case}_{ternary}"] = pb
    # gemm_lowbit
    for mode in (BNN, TNN, TBN):
        da, db = mode_dists(mode)
        for case, (m, n, k) in enumerate(SMALL_GEMM):
            seed = 2000 + 100 * mode + case
            if k == 32767:  # depth-contract golden: all +1 -> all 32767 (test_gemm.cpp:95-99)
                if mode != BNN:
                    continue
                a = np.ones((m, k), np.int8)
                b = np.ones((k, n), np.int8)
            else:
                a = port.generate(da, seed, 0, m, k)
                b = port.generate(db, seed, 1, k, n)
            for k_blk in ((4096, 64) if k < 32767 else (4096,)):
                c = ref.gemm(mode, a, b, k_blk)
                out[f"gemm_{mode}_{case}_{k_blk}"] = c
    # conv2d_lowbit (conv.cpp:33-59)
    conv_cases = [(5, 5, 2, 3, 3, 2, 1, 3), (8, 8, 5, 3, 3, 1, 1, 4), (9, 9, 32, 1, 1, 2, 0, 4),
                  (3, 3, 2, 3, 3, 1, 1, 2), (6, 7, 3, 3, 3, 1, 0, 5)]
    for mode in (BNN, TNN, TBN):
        da, db = mode_dists(mode)
        for case, (h, w, ch, kh, kw, s, p, cout) in enumerate(conv_cases):
            seed = 3000 + 100 * mode + case
            fm = port.generate(da, seed, 0, h * w, ch).reshape(h, w, ch)
            wt = port.generate(db, seed, 1, kh * kw * ch, cout)
            for pad_value in ((1, -1) if mode == BNN else (1,)):
                r = ref.conv2d_lowbit(mode, fm, mode == BNN, wt, mode != TNN, kh, kw, s, p, pad_value)
                out[f"conv_{mode}_{case}_{pad_value}"] = r
    return out


def config1(port, ref):
    a = port.generate(UNI3, 43, 0, 360, 256)
    b = port.generate(UNI3, 43, 1, 256, 96)
    return ref.gemm(TNN, a, b)


def config2(port, ref):
    outs = []
    for s, (m, n, k) in enumerate(sweep_shapes()):
        a = port.generate(SPARSE3, 44, 2 * s, m, k)
        b = port.generate(PM1, 44, 2 * s + 1, k, n)
        outs.append(ref.gemm(TBN, a, b))
    return outs


def big_gemm_hash(port, ref, mode, seed, m, n, k, dist_a, dist_b, chunk=65536, threads=None):
    threads = threads or os.cpu_count()
    b = port.generate(dist_b, seed, 1, k, n)
    b0, b1 = ref.encode(b, b_mode_ternary(mode))
    h = hashlib.sha256()
    for r0 in range(0, m, chunk):
        rows = min(chunk, m - r0)
        a = port.generate(dist_a, seed, 0, rows, k, row0=r0)
        a0, a1 = ref.encode(a, a_mode_ternary(mode))
        hd = ref.bench_prepare(mode, a0, a1, rows, k, b0, b1, n, threads)
        c = np.empty((rows, n), np.int16)
        ref.bench_run(hd, c)
        ref.bench_free(hd)
        h.update(np.ascontiguousarray(c, "<i2").tobytes())
        print(f"  rows {r0 + rows}/{m}", flush=True)
    return h.hexdigest()


def config4_hash(port, ref):
    # NHWC batch 64 x 56 x 56 x 128, 3x3x128 -> 128, stride 1, pad 1; one image per reference call
    h = hashlib.sha256()
    wt = port.generate(UNI3, 46, 1, 3 * 3 * 128, 128)
    for img in range(64):
        fm = port.generate(UNI3, 46, 0, 56 * 56, 128, row0=img * 56 * 56).reshape(56, 56, 128)
        r = ref.conv2d_lowbit(TNN, fm, False, wt, False, 3, 3, 1, 1)
        h.update(np.ascontiguousarray(r.astype(np.int16), "<i2").tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also hash configs 3-5 (minutes of CPU)")
    args = ap.parse_args()
    port, ref = Port(), Ref()
    t0 = time.time()
    small = make_small(port, ref)
    c1 = config1(port, ref)
    small["config1"] = c1
    c2 = config2(port, ref)
    for s, c in enumerate(c2):
        small[f"config2_{s}"] = c
    np.savez_compressed(SMALL, **small)
    meta = json.load(open(CONFIGS)) if os.path.exists(CONFIGS) else {}
    meta["generator"] = "splitmix64(seed ^ matrix_id<<56 ^ (row*cols+col)); A=matrix 0, B=matrix 1"
    meta["hash"] = "sha256 of int16 C, row-major little-endian"
    meta["c1"] = {"mode": "tnn", "m": 360, "n": 96, "k": 256, "seed": 43, "dist_a": UNI3, "dist_b": UNI3,
                  "sha256": sha(c1)}
    meta["c2"] = {"mode": "tbn", "seed": 44, "dist_a": SPARSE3, "dist_b": PM1,
                  "matrix_ids": "A=2*s, B=2*s+1 for shape index s (M-major, then N, then K)",
                  "sha256": [sha(c) for c in c2]}
    print(f"small fixtures done in {time.time() - t0:.1f}s", flush=True)
    if args.big:
        t = time.time()
        meta["c3"] = {"mode": "bnn", "m": 8192, "n": 8192, "k": 4096, "seed": 45, "dist_a": PM1, "dist_b": PM1,
                      "sha256": big_gemm_hash(port, ref, BNN, 45, 8192, 8192, 4096, PM1, PM1, chunk=2048)}
        print(f"c3 {time.time() - t:.1f}s", flush=True)
        t = time.time()
        meta["c4"] = {"mode": "tnn", "batch": 64, "h": 56, "w": 56, "c": 128, "kh": 3, "kw": 3, "stride": 1,
                      "pad": 1, "cout": 128, "seed": 46, "dist_fm": UNI3, "dist_w": UNI3,
                      "fm_rows": "image b, pixel (y,x) = generator row b*3136 + y*56 + x, 128 cols",
                      "sha256": config4_hash(port, ref)}
        print(f"c4 {time.time() - t:.1f}s", flush=True)
        t = time.time()
        meta["c5"] = {"mode": "tnn", "m": 1048576, "n": 1024, "k": 2048, "seed": 47, "dist_a": UNI3,
                      "dist_b": UNI3,
                      "sha256": big_gemm_hash(port, ref, TNN, 47, 1048576, 1024, 2048, UNI3, UNI3, chunk=65536)}
        print(f"c5 {time.time() - t:.1f}s", flush=True)
    with open(CONFIGS, "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
