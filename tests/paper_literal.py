"""Independent pure-Python pins for the oracle (test helpers; no shared code with oracle/ or
the CUDA path).  Each function transcribes the paper's own algorithm LITERALLY (not the
definitions the oracle uses), so agreement on many inputs pins the oracle.

  alg1_pruf            Alg. 1: step I, Sync step II with S' buffer,
                       step III with reduction rate RR and frozen reads per global
                       iteration, step IV Union/Find with min-root.
  alg3_balanced        Alg. 3 tile emulation: in-block iterations on a private
                       copy with a frozen 1-pixel band per global iteration.
  step3_iterations     step III iteration count on a chain (Fig. 4).
  kruskal_waterfall    O8: Kruskal MST under K, then per level each component takes its
                       min-K TREE edge (the classical waterfall = watershed on the MST of
                       the RAG).
  level1_by_partner    brute-force newmin (Alg. 4 l.1-7) + "largest-label
                       neighbour among the lowest passes" partner rule (Eq. 1 transposed).
  count_regional_minima  flood fill of minimal plateaux.
"""
from __future__ import annotations

import itertools
from collections import deque

import numpy as np


def neighbour_table(shape, conn, ndim):
    """N(p) for every p (clipped borders, p excluded; 2D images are independent
    along axis 0).  Lists are in increasing linear-index order."""
    n0, n1, n2 = shape
    offs = []
    zr = (-1, 0, 1) if ndim == 3 else (0,)
    for dz, dy, dx in itertools.product(zr, (-1, 0, 1), (-1, 0, 1)):
        if (dz, dy, dx) == (0, 0, 0):
            continue
        if conn in (4, 6) and abs(dz) + abs(dy) + abs(dx) != 1:
            continue
        offs.append((dz, dy, dx))
    table = []
    for z in range(n0):
        for y in range(n1):
            for x in range(n2):
                nb = []
                for dz, dy, dx in offs:
                    zz, yy, xx = z + dz, y + dy, x + dx
                    if 0 <= zz < n0 and 0 <= yy < n1 and 0 <= xx < n2:
                        nb.append((zz * n1 + yy) * n2 + xx)
                table.append(sorted(nb))
    return table


def canonical(L):
    """Relabel a partition so each label is the smallest index of its class (C7)."""
    L = list(L)
    first = {}
    for p, l in enumerate(L):
        first.setdefault(l, p)
    return [first[l] for l in L]


def alg1_pruf(I, nbrs, RR=6, trace=None):
    """Literal Alg. 1 (PRUF, Sync).  Returns final L (raw roots).  ``trace`` (dict) receives
    states after step I, step II iteration count, S/L after step II, step III count."""
    N = len(I)
    L = [0] * N
    S = [0] * N
    for p in range(N):  # Step I (l.1-10)
        nb = nbrs[p]
        if not nb:
            L[p], S[p] = p, 1
            continue
        m = min(I[r] for r in nb)
        q = max(r for r in nb if I[r] == m)  # Eq. 1
        if I[q] < I[p]:
            L[p], S[p] = q, 0
        elif I[q] > I[p]:
            L[p], S[p] = p, 1
        elif q > p:
            L[p], S[p] = q, 2
        else:
            L[p], S[p] = p, 3
    if trace is not None:
        trace["S1"] = list(S)
    it2 = 0
    while True:  # Step II (l.11-18): read S, write S' (Jacobi), swap
        it2 += 1
        change = False
        S2 = list(S)
        for p in range(N):
            if S[p] >= 2:
                cand = [q for q in nbrs[p] if S[q] == 0 and I[q] == I[p]]
                if cand:
                    L[p] = max(cand)  # C5: max index among the candidates
                    S2[p] = 0
                    change = True
        S = S2
        if trace is not None:
            trace.setdefault("S2_hist", []).append(list(S))
        if not change:
            break
    if trace is not None:
        trace["it2"] = it2
        trace["S2"] = list(S)
        trace["L2"] = list(L)
    it3 = 0
    while True:  # Step III (l.19-23): RR jumps per global sync, frozen reads
        it3 += 1
        Lold = list(L)
        for p in range(N):
            l = Lold[p]
            for _ in range(RR):
                if l == Lold[l]:
                    break
                l = Lold[l]
            L[p] = l
        if L == Lold:
            break
    if trace is not None:
        trace["it3"] = it3

    def find(x):
        while L[x] != x:
            x = L[x]
        return x

    for p in range(N):  # Step IV (l.24-27): Union over q > p, both S >= 2
        if S[p] >= 2:
            for q in nbrs[p]:
                if q > p and S[q] >= 2:
                    rp, rq = find(p), find(q)
                    if rp != rq:  # min-root union
                        L[max(rp, rq)] = min(rp, rq)
    return [find(p) for p in range(N)]  # l.28-29 Find


def alg3_balanced(I, block, max_global=1000):
    """Alg. 3 on a 1-D image split into blocks of ``block`` pixels (P:510-541 example).
    Returns the list of state arrays after each global iteration (until no change)."""
    N = len(I)
    nbrs = [[q for q in (p - 1, p + 1) if 0 <= q < N] for p in range(N)]
    S = [0] * N
    for p in range(N):  # step I states
        m = min(I[r] for r in nbrs[p])
        q = max(r for r in nbrs[p] if I[r] == m)
        S[p] = 0 if I[q] < I[p] else 1 if I[q] > I[p] else (2 if q > p else 3)
    hist = []
    for _ in range(max_global):
        frozen = list(S)  # the band outside each block keeps the last global values
        new = list(S)
        for b0 in range(0, N, block):
            loc = {p: frozen[p] for p in range(max(0, b0 - 1), min(N, b0 + block + 1))}
            while True:  # in-block iterations until no block change (l.4-12)
                snap = dict(loc)  # SharedToLocal after SyncThreads: Jacobi inside the block
                ch = False
                for p in range(b0, min(N, b0 + block)):
                    best = None
                    for q in nbrs[p]:  # l.7: (S(p)>=2 and S(q)<=0) or S(p)+1 < S(q) <= 0
                        if I[q] == I[p] and snap[q] <= 0:
                            if (snap[p] >= 2 or snap[p] + 1 < snap[q]) and (best is None or snap[q] > best):
                                best = snap[q]
                    if best is not None:
                        loc[p] = best - 1  # l.8: S(p) := S(q) - 1
                        ch = True
                if not ch:
                    break
            for p in range(b0, min(N, b0 + block)):
                new[p] = loc[p]
        hist.append(new)
        if new == S:
            break
        S = new
    return hist


def step3_iterations(length, RR):
    """Changing global iterations of step III on one chain of ``length`` pixels."""
    L = [max(0, p - 1) for p in range(length)]
    changing = 0
    while True:
        Lold = list(L)
        for p in range(length):
            l = Lold[p]
            for _ in range(RR):
                if l == Lold[l]:
                    break
                l = Lold[l]
            L[p] = l
        if L == Lold:
            return changing
        changing += 1


def rag_bruteforce(labels, I, nbrs):
    """{(a,b): min height} over adjacent pairs with different labels (Alg. 4)."""
    E = {}
    for p in range(len(I)):
        for q in nbrs[p]:
            if labels[p] != labels[q]:
                a, b = min(labels[p], labels[q]), max(labels[p], labels[q])
                h = max(I[p], I[q])
                E[(a, b)] = min(E[(a, b)], h) if (a, b) in E else h
    return E


def _K(e):
    (a, b), w = e
    return (w, -b, -a)  # C14: w asc, max desc, min desc


def kruskal_waterfall(labels, I, nbrs, NL):
    """O8: levels[k] as canonical labels, via the MST of the RAG."""
    E = sorted(rag_bruteforce(labels, I, nbrs).items(), key=_K)
    reps = sorted(set(labels))
    par = {r: r for r in reps}

    def find(x):
        while par[x] != x:
            x = par[x]
        return x

    mst = []
    for (a, b), w in E:  # Kruskal
        ra, rb = find(a), find(b)
        if ra != rb:
            par[max(ra, rb)] = min(ra, rb)
            mst.append(((a, b), w))
    comp = {r: r for r in reps}
    levels = [list(labels)]
    for _ in range(1, NL):
        pick = {}
        for (a, b), w in mst:  # mst is in K order: first hit = min-K tree edge
            ca, cb = comp[a], comp[b]
            if ca == cb:
                continue
            pick.setdefault(ca, (a, b))
            pick.setdefault(cb, (a, b))
        par2 = {c: c for c in set(comp.values())}

        def f2(x):
            while par2[x] != x:
                x = par2[x]
            return x

        for (a, b) in pick.values():
            ra, rb = f2(comp[a]), f2(comp[b])
            if ra != rb:
                par2[max(ra, rb)] = min(ra, rb)
        comp = {r: f2(comp[r]) for r in reps}
        levels.append([comp[l] for l in labels])
    return levels


def level1_by_partner(labels, I, nbrs):
    """Level 1 from first principles: newmin(r) by the brute-force double loop of Alg. 4
    l.1-7 (M = 256 sentinel), partner(r) = the largest-label neighbouring region among those
    whose pass height equals newmin(r); level-1 regions = connected components of
    {r - partner(r)}; label = smallest member."""
    E = rag_bruteforce(labels, I, nbrs)
    newmin = {}
    for p in range(len(I)):
        for q in nbrs[p]:
            if labels[q] != labels[p]:
                h = max(I[p], I[q])
                newmin[labels[p]] = min(newmin.get(labels[p], 256), h)
    reps = sorted(set(labels))
    par = {r: r for r in reps}

    def find(x):
        while par[x] != x:
            x = par[x]
        return x

    for r in reps:
        if r not in newmin:
            continue
        partners = [b if a == r else a for (a, b), w in E.items() if r in (a, b) and w == newmin[r]]
        s = max(partners)
        ra, rb = find(r), find(s)
        if ra != rb:
            par[max(ra, rb)] = min(ra, rb)
    return [find(l) for l in labels]


def count_regional_minima(I, nbrs):
    """Number of minimal plateaux (equal-intensity components with no lower neighbour)."""
    N = len(I)
    seen = [False] * N
    count = 0
    for s in range(N):
        if seen[s]:
            continue
        comp = [s]
        seen[s] = True
        dq = deque([s])
        while dq:
            p = dq.popleft()
            for q in nbrs[p]:
                if not seen[q] and I[q] == I[p]:
                    seen[q] = True
                    comp.append(q)
                    dq.append(q)
        if not any(I[q] < I[p] for p in comp for q in nbrs[p]):
            count += 1
    return count


def as_list(a):
    return [int(v) for v in np.asarray(a).ravel()]
