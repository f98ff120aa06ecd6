"""Staircase decision plan restated on the CPU — TEST ORACLE ONLY.

Builds, with numpy and plain Python, the byte image that the device plan builders
(paper_2102_01887_b200/csrc/sp_plan.cu, sp_plan_cluster.cu) write for a (table, alpha), so that
the GPU builders are checked section by section against an independent restatement and the
decision kernels' input is pinned.  What the image encodes is the reference's argmin
(configurator.py:219-237) precomputed over every slack threshold:

* cost = ((res*lat)*price)/batch, costpen = cost + alpha*((lat*res)/(batch*pool))
  (configurator.py:224-226);
* argmin key (score, cost, res, id_rank) (configurator.py:229-237), score = cost on the feasible
  side (lat < slack) and costpen on the penalized side;
* per kind, positions in (lat, index) order; at every latency boundary p the per-batch-lane
  best feasible entry (prefix minimum over positions < p) and best penalized entry (suffix
  minimum over positions >= p); a row per boundary whose lane vector changed;
* candidates (entries that are some row's lane best) in one id space ordered by
  (score, cost, res, id_rank), feasible side first on exact ties; each row stores, for every
  lane interval [lo, hi], the minimum candidate id over its lanes.

``plan_image(...)`` returns a dict of named sections (numpy arrays) plus the header fields.
"""
from __future__ import annotations

import numpy as np

K_MAX_BUCKETS = 4096
K_MAX_LUT = 4097
HDR_BYTES = 512
NONE16 = 0xFFFF


def _hi(x: float) -> int:
    """__double2hiint reinterpreted as u32."""
    return int(np.array([x], dtype=np.float64).view(np.uint64)[0] >> np.uint64(32))


def _order_key(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float64).view(np.uint64)
    neg = (u >> np.uint64(63)) != 0
    return np.where(neg, ~u, u | np.uint64(1 << 63))


def plan_image(lat, res, batch, pool, price, kind, id_rank, K: int, alpha: float) -> dict:
    lat = np.asarray(lat, dtype=np.float64)
    res = np.asarray(res, dtype=np.float64)
    batch = np.asarray(batch, dtype=np.int64)
    pool = np.asarray(pool, dtype=np.float64)
    price = np.asarray(price, dtype=np.float64)
    kind = np.asarray(kind, dtype=np.int64)
    id_rank = np.asarray(id_rank, dtype=np.int64)
    M = len(lat)
    bvals = sorted(set(int(b) for b in batch))
    nB = len(bvals)
    lane = np.searchsorted(np.array(bvals), batch)
    # configurator.py:224-225 in numpy order
    cost = ((res * lat) * price) / batch.astype(np.float64)
    costpen = cost + alpha * ((lat * res) / (batch.astype(np.float64) * pool))
    # r1: rank under (cost, res, id_rank); r2: rank under (costpen, r1)
    o1 = np.lexsort((id_rank, res, cost))
    r1 = np.empty(M, np.int64)
    r1[o1] = np.arange(M)
    o2 = np.lexsort((r1, costpen))
    r2 = np.empty(M, np.int64)
    r2[o2] = np.arange(M)
    INF = np.iinfo(np.int64).max
    kinds = []
    candf, cands = set(), set()
    for k in range(K):
        ents = np.flatnonzero(kind == k)
        if len(ents) == 0:
            kinds.append(None)
            continue
        ok = _order_key(lat[ents])
        pos = ents[np.lexsort((ents, ok))]  # (lat, index) order
        Mk = len(pos)
        # PF[b][p] = min r1 over positions < p in lane b; PS[b][p] = min r2 over positions >= p
        PF = np.full((nB, Mk + 1), INF, np.int64)
        PS = np.full((nB, Mk + 1), INF, np.int64)
        run = np.full(nB, INF, np.int64)
        for p in range(Mk):
            PF[:, p] = run
            e = pos[p]
            run[lane[e]] = min(run[lane[e]], r1[e])
        PF[:, Mk] = run
        run = np.full(nB, INF, np.int64)
        for p in range(Mk - 1, -1, -1):
            e = pos[p]
            run[lane[e]] = min(run[lane[e]], r2[e])
            PS[:, p] = run
        rows, thr = [], []
        prev = None
        for p in range(Mk + 1):
            isb = p == 0 or p == Mk or lat[pos[p]] != lat[pos[p - 1]]
            if not isb:
                continue
            vec = (tuple(PF[:, p]), tuple(PS[:, p]))
            if p == 0 or vec != prev:
                rows.append(vec)
                thr.append(-np.inf if p == 0 else lat[pos[p - 1]])
                for v in vec[0]:
                    if v != INF:
                        candf.add(int(v))
                for v in vec[1]:
                    if v != INF:
                        cands.add(int(v))
            prev = vec
        kinds.append((rows, np.array(thr)))
    # unified candidate ids: CP (feasible, by r1) and CS (penalized, by r2) merged by
    # (score, r1), CP first on ties
    cp = sorted(candf)                       # r1 ranks
    cs = sorted(cands)                       # r2 ranks
    cp_ent = [int(o1[r]) for r in cp]
    cs_ent = [int(o2[r]) for r in cs]
    keys = [(cost[e], r1[e], 0, i) for i, e in enumerate(cp_ent)] + \
           [(costpen[e], r1[e], 1, i) for i, e in enumerate(cs_ent)]
    keys.sort()
    uid_cp, uid_cs = {}, {}
    for u, (_, _, side, i) in enumerate(keys):
        (uid_cp if side == 0 else uid_cs)[i] = u
    cp_pos = {r: i for i, r in enumerate(cp)}
    cs_pos = {r: i for i, r in enumerate(cs)}
    ncp, ncs = len(cp), len(cs)
    n = ncp + ncs
    score = np.empty(n)
    clat = np.empty(n)
    meta = np.empty(n, np.uint32)
    cbatch = np.empty(n, np.int32)
    for i, e in enumerate(cp_ent):
        u = uid_cp[i]
        score[u], clat[u] = cost[e], lat[e]
        meta[u] = e | (1 << 16) | (int(kind[e]) << 17)
        cbatch[u] = batch[e]
    for i, e in enumerate(cs_ent):
        u = uid_cs[i]
        score[u], clat[u] = costpen[e], lat[e]
        meta[u] = e | (int(kind[e]) << 17)
        cbatch[u] = batch[e]
    nq = nB * (nB + 1) // 2
    out = {"M": M, "nB": nB, "K": K, "ncp": ncp, "ncs": ncs, "batch_vals": bvals,
           "row_stride": ((nB * (nB + 1) + 3) // 4) * 4, "score": score, "lat": clat,
           "meta": meta, "batch": cbatch, "kinds": []}
    maxB = max(bvals)
    out["lut_n"] = maxB + 2 if maxB + 2 <= K_MAX_LUT else 0
    bv = np.array(bvals)
    out["lut"] = np.array([int((bv < v).sum()) | (int((bv <= v).sum()) << 8) for v in range(out["lut_n"])],
                          dtype=np.uint16)
    for k in range(K):
        if kinds[k] is None:
            out["kinds"].append({"R": 0})
            continue
        rows, thr = kinds[k]
        R = len(rows)
        lanes = np.empty((R, nB), np.int64)
        for r, (pf, ps) in enumerate(rows):
            for b in range(nB):
                a = uid_cp[cp_pos[pf[b]]] if pf[b] != INF else INF
                s = uid_cs[cs_pos[ps[b]]] if ps[b] != INF else INF
                lanes[r, b] = min(a, s)
        enc = np.empty((R, nq), np.uint16)
        q = 0
        for lo in range(nB):
            for hi in range(lo, nB):
                m = lanes[:, lo:hi + 1].min(axis=1)
                enc[:, q] = np.where(m == INF, NONE16, m)
                q += 1
        nbk, shift, kmin, generic = 1, 0, 0, 0
        if R >= 2:
            kmin = _hi(thr[1])
            kmax = _hi(thr[R - 1])
            while nbk < 2 * (R - 1) and nbk < K_MAX_BUCKETS:
                nbk <<= 1
            while ((kmax - kmin) & 0xFFFFFFFF) >> shift >= nbk:
                shift += 1
            generic = int(not (thr[1] > 0.0))
        cnt = np.zeros(nbk, np.int64)
        for j in range(1, R):
            b = min((((_hi(thr[j]) - kmin) & 0xFFFFFFFF) >> shift), nbk - 1)
            cnt[b] += 1
        below = np.concatenate([[0], np.cumsum(cnt)[:-1]])
        bkt = (below | (cnt << 16)).astype(np.uint32)
        out["kinds"].append({"R": R, "thr": thr, "rows": enc, "kmin_hi": kmin,
                             "nb1_shift": (nbk - 1) | (shift << 16), "generic": generic,
                             "bkt": bkt})
    return out


def parse_image(img: bytes | np.ndarray) -> dict:
    """Sections of a device plan image (same layout as plan_image's output)."""
    b = np.frombuffer(bytes(img), dtype=np.uint8)
    i32 = b[:HDR_BYTES].view(np.int32)
    u32 = b[:HDR_BYTES].view(np.uint32)
    out = {"magic": int(u32[0]), "total_bytes": int(i32[1]), "M": int(i32[2]), "nB": int(i32[3]),
           "W": int(i32[4]), "K": int(i32[5]), "ncp": int(i32[6]), "ncs": int(i32[7]),
           "row_stride": int(i32[11]), "lut_n": int(i32[13])}
    score_off, lat_off, recb_off, lut_off = int(i32[8]), int(i32[9]), int(i32[10]), int(i32[12])
    out["batch_vals"] = [int(x) for x in i32[16:16 + out["nB"]]]
    n = out["ncp"] + out["ncs"]
    out["score"] = b[score_off:score_off + 8 * n].view(np.float64)
    out["lat"] = b[lat_off:lat_off + 8 * n].view(np.float64)
    rec = b[recb_off:recb_off + 8 * n].view(np.uint32).reshape(-1, 2)
    out["meta"] = rec[:, 0].copy()
    out["batch"] = rec[:, 1].view(np.int32).copy()
    out["lut"] = b[lut_off:lut_off + 2 * out["lut_n"]].view(np.uint16)
    nq = out["nB"] * (out["nB"] + 1) // 2
    out["kinds"] = []
    for k in range(8):
        d = b[128 + 32 * k: 128 + 32 * (k + 1)]
        du, di = d.view(np.uint32), d.view(np.int32)
        R = int(di[5])
        if k >= out["K"]:
            continue
        if R == 0:
            out["kinds"].append({"R": 0})
            continue
        thr = b[int(di[2]):int(di[2]) + 8 * R].view(np.float64)
        rows = np.stack([b[int(di[3]) + r * out["row_stride"]: int(di[3]) + r * out["row_stride"] + 2 * nq]
                         .view(np.uint16) for r in range(R)])
        nbk = (int(du[1]) & 0xFFFF) + 1
        out["kinds"].append({"R": R, "thr": thr, "rows": rows, "kmin_hi": int(du[0]),
                             "nb1_shift": int(du[1]), "generic": int(di[6]),
                             "bkt": b[int(di[4]):int(di[4]) + 4 * nbk].view(np.uint32)})
    return out


def compare(a: dict, b: dict) -> list[str]:
    """Names of the sections where two parsed images differ (empty when identical)."""
    bad = []
    for key in ("M", "nB", "K", "ncp", "ncs", "row_stride", "lut_n", "batch_vals"):
        if a[key] != b[key]:
            bad.append(key)
    for key in ("score", "lat"):
        if not np.array_equal(np.asarray(a[key]).view(np.uint64), np.asarray(b[key]).view(np.uint64)):
            bad.append(key)
    for key in ("meta", "batch", "lut"):
        if not np.array_equal(np.asarray(a[key]), np.asarray(b[key])):
            bad.append(key)
    for k, (x, y) in enumerate(zip(a["kinds"], b["kinds"])):
        if x["R"] != y["R"]:
            bad.append(f"kind{k}.R")
            continue
        if x["R"] == 0:
            continue
        if not np.array_equal(np.asarray(x["thr"]).view(np.uint64), np.asarray(y["thr"]).view(np.uint64)):
            bad.append(f"kind{k}.thr")
        if not np.array_equal(x["rows"], y["rows"]):
            bad.append(f"kind{k}.rows")
        for key in ("kmin_hi", "nb1_shift", "generic"):
            if x[key] != y[key]:
                bad.append(f"kind{k}.{key}")
        if not np.array_equal(x["bkt"], y["bkt"]):
            bad.append(f"kind{k}.bkt")
    return bad


def plan_argmin(img: dict, slack, min_lane: int, excluded_mask: int = 0):
    """The argmin a decision kernel reads from a plan (no delay / downgrade): per kind the row
    of the last threshold below the slack, the lane interval [min_lane, nB-1], the minimum
    candidate id over the kinds not excluded.  Returns (entry, feasible) or None."""
    nB = img["nB"]
    best = NONE16
    for k, kd in enumerate(img["kinds"]):
        if kd["R"] == 0 or (excluded_mask >> k) & 1 or min_lane >= nB:
            continue
        r = int(np.searchsorted(kd["thr"], slack[k], side="left")) - 1  # last thr < slack
        q = min_lane * nB - (min_lane * (min_lane - 1)) // 2 + (nB - 1 - min_lane)
        best = min(best, int(kd["rows"][r, q]))
    if best == NONE16:
        return None
    m = int(img["meta"][best])
    return m & 0x7FFF, bool((m >> 16) & 1)
