#!/usr/bin/env python
"""NumPy simulation of K1g rounds on one uniform cloud (kd buckets of 32, KM = 16):
the ordered chain test, then (below the threshold P0) a continuation that picks
the remaining candidates by their updated values and accepts while the pick
beats every other candidate, every non-key point (second best / triangle
bound from each winner) and every unlisted bucket.  Prints rounds and checks
the winners against exact FPS.  Usage: python tools/sim_chain_continuation.py N P0"""
rng = np.random.default_rng(0)
n = int(sys.argv[1]); iters = n // 4
P = rng.random((n, 3)).astype(np.float32)
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
box = np.array([np.concatenate([P[l].min(0), P[l].max(0)]) for l in leaves], np.float32)
def d2(a, p):
    d = (a - p).astype(np.float32)
    return ((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2]).astype(np.float32)
def fc(p, bq):
    lo = np.abs((bq[:, :3] - p).astype(np.float32)); hi = np.abs((bq[:, 3:] - p).astype(np.float32))
    g = np.maximum(lo, hi)
    return ((g[:, 0] * g[:, 0] + g[:, 1] * g[:, 1]) + g[:, 2] * g[:, 2]).astype(np.float32)
KM = 16
P0 = int(sys.argv[2]) if len(sys.argv) > 2 else 17
dist = np.full(n, np.inf, np.float32)
sel = [0]; newpts = [0]
rounds = 0; hist = []; steps = 0; cont_rounds = 0
while len(sel) < iters:
    for s in newpts:
        dist = np.minimum(dist, d2(P, P[s]))
    dist[np.array(sel)] = -np.inf
    order = np.lexsort((np.arange(n), -dist.astype(np.float64), bid))
    starts = np.searchsorted(bid[order], np.arange(nb))
    ends = np.append(starts[1:], n)
    key = order[starts]
    sec = np.where(ends - starts > 1, dist[order[np.minimum(starts + 1, n - 1)]], -np.inf).astype(np.float32)
    kv = dist[key]
    rk = np.lexsort((key, -kv.astype(np.float64)))[:KM]
    c = key[rk]; cv = kv[rk]; c2 = sec[rk]; cb = box[rk]; cpos = c
    rself = np.array([fc(P[c[i]], cb[i:i+1])[0] for i in range(KM)])
    tb = np.minimum(c2, rself)
    acc = [0]
    for j in range(1, KM):
        ok = cv[j] >= 0
        for i in range(j):
            if d2(P[c[j]], P[c[i]]) < cv[j] or not (cv[j] > tb[i]): ok = False; break
        if not ok: break
        acc.append(j)
    p = len(acc)
    if p < KM and p < P0 and len(sel) + p < iters:
        cont_rounds += 1
        alive = np.ones(KM, bool); alive[:p] = False
        u = cv.copy()
        for a in acc: u = np.minimum(u, d2(P[c], P[c[a]]))
        ob = c2.copy().astype(np.float64)   # other points of B_j: <= sec_j
        ob[:p] = tb[:p]
        sr = np.sqrt(rself.astype(np.float64))
        def ub(w):  # triangle bound of d2(x, c_w), x in B_j
            return (sr + np.sqrt(d2(P[c], P[c[w]]).astype(np.float64))) ** 2 * (1 + 1e-6)
        for a in acc: ob = np.where(alive, np.minimum(ob, ub(a)), ob)
        while alive.any():
            steps += 1
            idx = np.flatnonzero(alive)
            w = idx[np.lexsort((cpos[idx], -u[idx].astype(np.float64)))[0]]
            uw = u[w]
            ok = uw >= 0 and np.all(uw > ob) and (uw > cv[-1] or (uw == cv[-1] and cpos[w] <= cpos[-1]))
            if not ok: break
            acc.append(w); alive[w] = False
            u = np.minimum(u, d2(P[c], P[c[w]]))
            ob = np.where(alive, np.minimum(ob, ub(w)), ob)
            ob[w] = min(ob[w], tb[w])
            if len(sel) + len(acc) >= iters: break
    accp = [c[a] for a in acc][:iters - len(sel)]
    sel += accp; newpts = accp; rounds += 1; hist.append(len(accp))
h = np.array(hist)
dd = np.full(n, np.inf, np.float32); ref = [0]; pp = 0
for it in range(1, iters):
    dd = np.minimum(dd, d2(P, P[pp])); dd[pp] = -np.inf
    pp = int(np.argmax(dd)); ref.append(pp)
bad = np.flatnonzero(np.array(sel[:iters]) != np.array(ref))
print("P0", P0, "n", n, "rounds", rounds, "winners/round", round(len(sel) / rounds, 2),
      "early", round(h[:len(h)//10].mean(), 2), "late", round(h[len(h)//10:].mean(), 2),
      "cont rounds", cont_rounds, "steps", steps, "exact", bad.size == 0, flush=True)
