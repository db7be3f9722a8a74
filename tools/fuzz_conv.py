"""Randomised conv2d_lowbit shapes (stride 1, c % 128 == 0: the halo kernels K7 / K7T, K6 when they do not fit)
against the oracle's conv2d_lowbit (im2col -> encode by sign -> GeMM, conv.cpp:33-59).  SECONDS of fuzzing, seeded; prints the failing shape if any."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_09120_b200 as lb
from oracle.oracle import Port, BNN, TNN, TBN
from tests.golden.make_golden import mode_dists

port = Port()
rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
t_end = time.time() + float(os.environ.get("SECONDS", "300"))
n = 0
paths = {}
while time.time() < t_end:
    mode = int(rng.choice([BNN, TNN, TBN]))
    ksz = int(rng.choice([1, 2, 3, 3, 3, 5]))
    pad = int(rng.integers(0, min(2, ksz - 1) + 1))
    ch = int(rng.choice([128, 128, 256, 384]))
    cout = int(rng.integers(1, 40)) * 8
    b = int(rng.integers(1, 5))
    h = int(rng.integers(max(1, ksz - 2 * pad), 14))
    w = int(rng.choice([rng.integers(max(1, ksz - 2 * pad), 34), rng.integers(30, 70), rng.integers(60, 160)]))
    binary = mode == BNN
    pv = int(rng.choice([1, -1])) if binary else int(rng.choice([1, -1, 0]))
    fm_binary = binary or (mode != BNN and rng.random() < 0.25)
    da, db = mode_dists(mode)
    seed = 1000 + n
    fm = port.generate(1 if fm_binary else da, seed, 0, b * h * w, ch).reshape(b, h, w, ch)
    if not fm_binary and rng.random() < 0.3:
        fm = (fm * np.int8(rng.choice([2, 3, 127]))).astype(np.int8)  # values mapped by sign
    wt = port.generate(db, seed, 1, ksz * ksz * ch, cout)
    bp = lb.encode_ternary(torch.from_numpy(wt).cuda()) if mode == TNN else lb.encode_binary(torch.from_numpy(wt).cuda())
    wts = lb.prepare_weights(lb.pack_b(bp))
    path = lb.conv_select(mode, fm_binary, b, h, w, ch, cout, ksz, ksz, 1, pad)
    paths[path] = paths.get(path, 0) + 1
    try:
        got = lb.conv2d_lowbit(mode, torch.from_numpy(fm).cuda(), fm_binary, wts, ksz, ksz, 1, pad,
                               binary_pad_value=pv).cpu().numpy()
    except Exception as ex:
        print("ERROR", dict(mode=mode, fm_binary=fm_binary, b=b, h=h, w=w, ch=ch, cout=cout, ksz=ksz, pad=pad, pv=pv,
                            seed=seed, path=path), repr(ex))
        sys.exit(1)
    for img in range(b):
        want = port.conv2d_lowbit(mode, fm[img], fm_binary, wt, mode != TNN, ksz, ksz, 1, pad, pv)
        if not (got[img].astype(np.int32) == want).all():
            print("MISMATCH", dict(mode=mode, fm_binary=fm_binary, b=b, h=h, w=w, ch=ch, cout=cout, ksz=ksz, pad=pad, pv=pv,
                                   seed=seed, img=img, path=path, bad=int((got[img].astype(np.int32) != want).sum())))
            sys.exit(1)
    n += 1
print(f"fuzz OK: {n} convs, paths {paths}")
