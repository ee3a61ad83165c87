#!/usr/bin/env python3
"""Offline model of the ring kernel's shared-memory table reads (no GPU).

Builds the ring plan of a Kuhn cube the way rings.cu does (Morton origin
order, 256-edge tiles, sorted-rank slots, lane-transposed steps) and counts
bank-conflict wavefronts of the per-step table reads under the sm_100 model:
LDS.128 in quarter-warp phases over 8 16-byte bank groups, LDS.64 in
half-warp phases over 16 8-byte bank pairs (same address = broadcast).
Used to evaluate slot assignments before spending GPU time.
"""
import argparse
import os
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00778_b200 import meshgen  # noqa: E402


def spread(v):
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    for sh, m in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                  (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        v = (v | (v << np.uint64(sh))) & np.uint64(m)
    return v


def build(n, amp=0.15, permute=False):
    m = meshgen.tet_cube(n, amp=amp)
    if permute:
        m = meshgen.permute(m)
    x = m.coords.reshape(-1, 3)
    el = m.elements.reshape(-1, 4).astype(np.int64)
    nv = x.shape[0]
    loc = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    a = np.stack([el[:, p] for p, _ in loc], 1)
    b = np.stack([el[:, q] for _, q in loc], 1)
    j, k = np.minimum(a, b), np.maximum(a, b)
    key = (j * nv + k).ravel()
    ukey = np.unique(key)
    edges = np.stack([ukey // nv, ukey % nv], 1)
    eid = np.searchsorted(ukey, key)
    tet = np.repeat(np.arange(el.shape[0]), 6)
    order = np.lexsort((tet, eid))
    inc_e, inc_t = eid[order], tet[order]
    ptr = np.searchsorted(inc_e, np.arange(len(ukey) + 1))
    # rings
    seqs = []
    for e in range(len(ukey)):
        jj, kk = edges[e]
        ab = []
        for q in range(ptr[e], ptr[e + 1]):
            o = [v for v in el[inc_t[q]] if v != jj and v != kk]
            ab.append(o)
        cnt = defaultdict(int)
        for p_, q_ in ab:
            cnt[p_] += 1
            cnt[q_] += 1
        once = [v for v, c in cnt.items() if c == 1]
        start = min(once) if once else ab[0][0]
        used = [False] * len(ab)
        cur, seq = start, [jj, kk, start]
        for _ in range(len(ab)):
            for i, (p_, q_) in enumerate(ab):
                if not used[i] and (p_ == cur or q_ == cur):
                    used[i] = True
                    cur = q_ if p_ == cur else p_
                    seq.append(cur)
                    break
        seqs.append(seq)
    # Morton order of origins -> edge permutation
    lo = x.min(0)
    ext = (x.max(0) - lo).max()
    q = np.clip(((x - lo) * (2097151.0 / ext)).astype(np.int64), 0, 2097151)
    mk = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
    morder = np.argsort(mk, kind="stable")
    rank = np.empty(nv, np.int64)
    rank[morder] = np.arange(nv)
    os_ = np.searchsorted(edges[:, 0], np.arange(nv + 1))
    eperm = np.concatenate([np.arange(os_[o], os_[o + 1]) for o in morder])
    return seqs, eperm, rank


def tiles(seqs, eperm, rank, T=256):
    """Per tile: list of per-position rank sequences and the sorted unique ranks."""
    out = []
    for t0 in range(0, len(eperm), T):
        rs = [[int(rank[v]) for v in seqs[e]] for e in eperm[t0:t0 + T]]
        u = sorted({r for s in rs for r in s})
        out.append((rs, u))
    return out


def wavefronts(rs, slot, lanes=32):
    """(xy LDS.128, z LDS.64, ideal xy, ideal z) wavefronts of one tile."""
    wxy = wz = ixy = iz = 0
    for w0 in range(0, len(rs), lanes):
        W = rs[w0:w0 + lanes]
        S = max(len(s) for s in W)
        for st in range(S):
            sl = [slot[s[st]] if st < len(s) else None for s in W]
            for qd in range(0, lanes, 8):
                g = defaultdict(set)
                for v in sl[qd:qd + 8]:
                    if v is not None:
                        g[v % 8].add(v)
                if g:
                    wxy += max(len(c) for c in g.values())
                    ixy += 1
            for hf in range(0, lanes, 16):
                g = defaultdict(set)
                for v in sl[hf:hf + 16]:
                    if v is not None:
                        g[v % 16].add(v)
                if g:
                    wz += max(len(c) for c in g.values())
                    iz += 1
    return wxy, wz, ixy, iz


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--permute", action="store_true")
    a = ap.parse_args()
    seqs, eperm, rank = build(a.n, permute=a.permute)
    T = tiles(seqs, eperm, rank)
    tot = np.zeros(4)
    nu = []
    for rs, u in T:
        slot = {r: i for i, r in enumerate(u)}
        tot += wavefronts(rs, slot)
        nu.append(len(u))
    print(f"tiles {len(T)} NU mean {np.mean(nu):.0f} max {max(nu)}")
    print(f"sorted slots: xy {tot[0]:.0f} (ideal {tot[2]:.0f}, x{tot[0]/tot[2]:.2f})  "
          f"z {tot[1]:.0f} (ideal {tot[3]:.0f}, x{tot[1]/tot[3]:.2f})")


if __name__ == "__main__":
    main()


def groups(rs, lanes=32):
    """Access groups of a tile: (phase width, distinct ranks) per warp step."""
    out = []
    for w0 in range(0, len(rs), lanes):
        W = rs[w0:w0 + lanes]
        S = max(len(s) for s in W)
        for st in range(S):
            r = [s[st] if st < len(s) else None for s in W]
            for ph in (8, 16):
                for q in range(0, lanes, ph):
                    d = sorted({v for v in r[q:q + ph] if v is not None})
                    if len(d) > 1:
                        out.append((ph, d))
    return out


def color_slots(rs, u, nslots=256, w8=1.0, w16=1.0, sweeps=2):
    """Greedy + local-search assignment of ranks to slots: node -> colour c
    (slot % 16), balancing capacity nslots / 16 per colour, minimising
    same-bank pairs in quarter-warp (mod 8) and half-warp (mod 16) groups."""
    idx = {r: i for i, r in enumerate(u)}
    n = len(u)
    W = defaultdict(float)  # (i, j, kind) pair weights
    adj = [defaultdict(lambda: [0.0, 0.0]) for _ in range(n)]
    for ph, d in groups(rs):
        ii = [idx[v] for v in d]
        k = 0 if ph == 8 else 1
        for a in range(len(ii)):
            for b in range(a + 1, len(ii)):
                adj[ii[a]][ii[b]][k] += 1
                adj[ii[b]][ii[a]][k] += 1
    cap = nslots // 16
    col = [-1] * n
    used = [0] * 16

    def cost(i, c):
        s = 0.0
        for j, (a8, a16) in adj[i].items():
            cj = col[j]
            if cj < 0:
                continue
            if cj == c:
                s += w8 * a8 + w16 * a16
            elif cj % 8 == c % 8:
                s += w8 * a8
        return s

    order = sorted(range(n), key=lambda i: -sum(a + b for a, b in adj[i].values()))
    for i in order:
        best = min((c for c in range(16) if used[c] < cap), key=lambda c: (cost(i, c), used[c]))
        col[i] = best
        used[best] += 1
    for _ in range(sweeps):
        for i in order:
            c0 = col[i]
            col[i] = -1
            used[c0] -= 1
            best = min((c for c in range(16) if used[c] < cap), key=lambda c: (cost(i, c), c != c0))
            col[i] = best
            used[best] += 1
    nxt = [0] * 16
    slot = {}
    for i in range(n):
        c = col[i]
        slot[u[i]] = c + 16 * nxt[c]
        nxt[c] += 1
    return slot


def compare(n, permute=False, nslots=256):
    seqs, eperm, rank = build(n, permute=permute)
    T = tiles(seqs, eperm, rank)
    a = np.zeros(4)
    b = np.zeros(4)
    for rs, u in T:
        a += wavefronts(rs, {r: i for i, r in enumerate(u)})
        b += wavefronts(rs, color_slots(rs, u, nslots))
    print(f"n={n} sorted: xy x{a[0]/a[2]:.2f} z x{a[1]/a[3]:.2f} | coloured({nslots}): "
          f"xy x{b[0]/b[2]:.2f} z x{b[1]/b[3]:.2f}")


def color_online(rs, u, nslots=256, lanes=32):
    """One pass over the tile's warp steps: each uncoloured node of a
    half-warp group takes the colour (slot % 16) least used in its half-warp
    group and its quarter-warp group (mod 8), capacity nslots / 16."""
    cap = nslots // 16
    col = {}
    used = [0] * 16
    for w0 in range(0, len(rs), lanes):
        W = rs[w0:w0 + lanes]
        S = max(len(s) for s in W)
        for st in range(S):
            r = [s[st] if st < len(s) else None for s in W]
            for h in range(0, lanes, 16):
                for lane in range(h, h + 16):
                    v = r[lane]
                    if v is None or v in col:
                        continue
                    q0 = lane - lane % 8
                    half = {x for x in r[h:h + 16] if x is not None and x in col}
                    quart = {x for x in r[q0:q0 + 8] if x is not None and x in col}
                    c16 = [0] * 16
                    for x in half:
                        c16[col[x]] += 1
                    c8 = [0] * 8
                    for x in quart:
                        c8[col[x] % 8] += 1
                    best = min((c for c in range(16) if used[c] < cap),
                               key=lambda c: (c16[c] + c8[c % 8], used[c]))
                    col[v] = best
                    used[best] += 1
    nxt = [0] * 16
    slot = {}
    for v in u:
        c = col[v]
        slot[v] = c + 16 * nxt[c]
        nxt[c] += 1
    return slot


def color_rank_bits(u, nslots=256, key=lambda r: r % 16):
    """Colour = a function of the Morton rank (no access analysis); full
    colour classes spill to the least used class."""
    cap = nslots // 16
    used = [0] * 16
    slot = {}
    for r in u:
        c = key(r)
        if used[c] >= cap:
            c = min(range(16), key=lambda q: used[q])
        slot[r] = c + 16 * used[c]
        used[c] += 1
    return slot


def refine(rs, u, slot, nslots=256, sweeps=1, lanes=32):
    """Min-conflict sweeps over nodes starting from an assignment `slot`
    (colour = slot % 16): each node moves to the colour with the fewest
    same-bank partners in the quarter (mod 8) and half (mod 16) groups it is
    read in."""
    cap = nslots // 16
    col = {r: slot[r] % 16 for r in u}
    used = [0] * 16
    for r in u:
        used[col[r]] += 1
    memb = defaultdict(list)  # node -> list of (half members, quarter members)
    for w0 in range(0, len(rs), lanes):
        W = rs[w0:w0 + lanes]
        S = max(len(s) for s in W)
        for st in range(S):
            r_ = [s[st] if st < len(s) else None for s in W]
            for h in range(0, lanes, 16):
                half = [x for x in r_[h:h + 16] if x is not None]
                for q in (h, h + 8):
                    quart = [x for x in r_[q:q + 8] if x is not None]
                    for x in set(quart):
                        memb[x].append((half, quart))
    for _ in range(sweeps):
        for v in u:
            c16 = [0] * 16
            c8 = [0] * 8
            for half, quart in memb[v]:
                for x in set(half):
                    if x != v:
                        c16[col[x]] += 1
                for x in set(quart):
                    if x != v:
                        c8[col[x] % 8] += 1
            used[col[v]] -= 1
            best = min((c for c in range(16) if used[c] < cap),
                       key=lambda c: (c16[c] + c8[c % 8], c != col[v]))
            col[v] = best
            used[best] += 1
    nxt = [0] * 16
    out = {}
    for r in u:
        c = col[r]
        out[r] = c + 16 * nxt[c]
        nxt[c] += 1
    return out


def refine_parallel(rs, u, slot, rounds=3, nslots=512, seed=0, lanes=32):
    """Jacobi-style min-conflict rounds (what a CTA can do in parallel): every
    node computes its best colour from the current colours; a node moves only
    if it improves and no co-member that also wants to move has a higher
    random priority.  Colour classes hold nslots / 16 slots."""
    rng = np.random.default_rng(seed)
    cap = nslots // 16
    col = {r: slot[r] % 16 for r in u}
    prio = {r: rng.random() for r in u}
    memb = defaultdict(list)
    for w0 in range(0, len(rs), lanes):
        W = rs[w0:w0 + lanes]
        S = max(len(s) for s in W)
        for st in range(S):
            r_ = [s[st] if st < len(s) else None for s in W]
            for h in range(0, lanes, 16):
                half = [x for x in r_[h:h + 16] if x is not None]
                for q in (h, h + 8):
                    quart = [x for x in r_[q:q + 8] if x is not None]
                    for x in set(quart):
                        memb[x].append((half, quart))
    for _ in range(rounds):
        used = [0] * 16
        for r in u:
            used[col[r]] += 1
        want = {}
        for v in u:
            c16 = [0] * 16
            c8 = [0] * 8
            for half, quart in memb[v]:
                for x in set(half):
                    if x != v:
                        c16[col[x]] += 1
                for x in set(quart):
                    if x != v:
                        c8[col[x] % 8] += 1
            cost = [c16[c] + c8[c % 8] for c in range(16)]
            b = min(range(16), key=lambda c: (cost[c], c != col[v]))
            if cost[b] < cost[col[v]]:
                want[v] = b
        for v, b in want.items():
            rivals = {x for half, _ in memb[v] for x in half
                      if x in want and x != v and want[x] % 8 == b % 8}
            if all(prio[v] > prio[x] for x in rivals) and used[b] < cap:
                used[col[v]] -= 1
                used[b] += 1
                col[v] = b
    nxt = [0] * 16
    out = {}
    for r in u:
        c = col[r]
        out[r] = c + 16 * nxt[c]
        nxt[c] += 1
    return out


def wavefronts_copies(rs, slot, ncopy=2, lanes=32, xor=(0, 4, 2, 6)):
    """Table with ncopy copies of every node (copy c of slot s at bank index
    s ^ xor[c]); each access picks a copy greedily per half warp so that the
    quarter (mod 8) and half (mod 16) phases see distinct banks where
    possible (same node -> same copy, a broadcast)."""
    wxy = wz = ixy = iz = 0
    for w0 in range(0, len(rs), lanes):
        W = rs[w0:w0 + lanes]
        S = max(len(s) for s in W)
        for st in range(S):
            sl = [slot[s[st]] if st < len(s) else None for s in W]
            phys = [None] * lanes
            for h in range(0, lanes, 16):
                chosen = {}
                for lane in range(h, h + 16):
                    v = sl[lane]
                    if v is None:
                        continue
                    if v in chosen:
                        phys[lane] = chosen[v]
                        continue
                    q0 = lane - lane % 8
                    best = None
                    for c in range(ncopy):
                        p = (v ^ xor[c]) + 256 * c
                        load16 = sum(1 for x in phys[h:h + 16] if x is not None and x % 16 == p % 16 and x != p)
                        load8 = sum(1 for x in phys[q0:q0 + 8] if x is not None and x % 8 == p % 8 and x != p)
                        key = (load8 + load16, c)
                        if best is None or key < best[0]:
                            best = (key, p)
                    phys[lane] = best[1]
                    chosen[v] = best[1]
            for qd in range(0, lanes, 8):
                g = defaultdict(set)
                for x in phys[qd:qd + 8]:
                    if x is not None:
                        g[x % 8].add(x)
                if g:
                    wxy += max(len(c) for c in g.values())
                    ixy += 1
            for hf in range(0, lanes, 16):
                g = defaultdict(set)
                for x in phys[hf:hf + 16]:
                    if x is not None:
                        g[x % 16].add(x)
                if g:
                    wz += max(len(c) for c in g.values())
                    iz += 1
    return wxy, wz, ixy, iz
