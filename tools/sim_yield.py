#!/usr/bin/env python
"""NumPy simulation of K1g's multi-winner rounds on one C5 FlashFPS cloud
(uniform 50K points, 12,500 winners, kd buckets of 32): rounds and winners per
round for each KM given on the command line (exact chain rule (a) + (b)).
Usage: python tools/sim_yield.py 16 32 64"""
import numpy as np, sys
rng = np.random.default_rng(0)
n = 50000; iters = 12500
P = rng.random((n, 3)).astype(np.float32)
# kd buckets of 32 points (median splits on longest axis)
def kd(idx, out):
    if len(idx) <= 32:
        out.append(idx); return
    pts = P[idx]; ax = np.argmax(pts.max(0) - pts.min(0))
    nl = ((len(idx) // 32 + 1) // 2) * 32
    o = np.argsort(pts[:, ax], kind='stable')
    kd(idx[o[:nl]], out); kd(idx[o[nl:]], out)
leaves = []; kd(np.arange(n), leaves)
bid = np.empty(n, np.int64)
for i, l in enumerate(leaves): bid[l] = i
nb = len(leaves)
def d2(a, p):
    d = a - p
    return (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
for KM in [int(x) for x in sys.argv[1:]]:
    dist = np.full(n, np.inf, np.float32)
    sel = [0]; dist[0] = -np.inf
    newpts = [0]
    rounds = 0; hist = []
    while len(sel) < iters:
        for s in newpts:
            dist = np.minimum(dist, d2(P, P[s])); dist[s] = -np.inf
        for s in sel[-len(newpts):]: dist[s] = -np.inf
        # bucket key (max, lowest pos) and second-best value
        order = np.lexsort((np.arange(n), -dist.astype(np.float64), bid))
        # order grouped by bucket, inside: value desc, pos asc
        starts = np.searchsorted(bid[order], np.arange(nb))
        key = order[starts]
        sec = dist[order[np.minimum(starts + 1, n - 1)]]
        kv = dist[key]
        rk = np.lexsort((key, -kv.astype(np.float64)))[:KM]
        acc = [key[rk[0]]]
        for j in range(1, KM):
            c = key[rk[j]]; ok = True
            for i in range(j):
                b = key[rk[i]]
                dd = d2(P[c:c+1], P[b])[0]
                if dd < dist[c] or not (dist[c] > sec[rk[i]]): ok = False; break
            if not ok: break
            acc.append(c)
        acc = acc[:iters - len(sel)]
        sel += acc; newpts = acc; rounds += 1; hist.append(len(acc))
    h = np.array(hist)
    print(KM, "rounds", rounds, "winners/round", len(sel) / rounds, "late", h[len(h)//10:].mean())
