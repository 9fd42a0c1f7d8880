"""Shared-memory bank-conflict model of the Stockham exchanges.

Counts wavefronts per warp-instruction for the writes and reads of every
pass, for the row layout (groups of TG threads, one transform each) and the
column layout (C transforms interleaved, thread tid = c + C*j).
Element size E bytes (8 fp32 complex, 16 fp64 complex): a warp access is
split into phases of 128/E threads; within a phase, each E-byte element
occupies E/4 consecutive banks; wavefronts = max over bank groups of the
number of distinct addresses hitting it.
"""
import itertools, sys
from collections import defaultdict

def shape(LG, LGR):
    lgR = min(LG, LGR); L = 1 << LG; R = 1 << lgR; TG = L // R
    NP = 0 if lgR == 0 else (LG + lgR - 1) // lgR
    lg_last = LG - (NP - 1) * lgR if NP else 0
    radix = lambda s: 1 << (lgR if s < NP - 1 else lg_last)
    return L, R, TG, NP, lgR, radix

def wavefronts(addrs, E):
    per_phase = 128 // E
    total = 0
    for p in range(0, 32, per_phase):
        grp = defaultdict(set)
        for a in addrs[p:p + per_phase]:
            if a is None: continue
            grp[(a // E) % (128 // E)].add(a)
        total += max((len(v) for v in grp.values()), default=0)
    return total

def simulate(LG, LGR, E, layout, C=1, colpad=2):
    L, R, TG, NP, lgR, radix = shape(LG, LGR)
    pad = lambda i: i + (i >> lgR)
    SM = L + (L >> lgR)
    S = SM + colpad
    nthreads = TG * C if layout == 'col' else max(TG, 32)
    def thread(tid):
        if layout == 'col': return tid % C, tid // C
        return tid // TG, tid % TG
    res = []
    for s in range(NP - 1):
        Rs = radix(s); Ns = R ** s; Q = R // Rs
        # writes
        w_total = w_ideal = 0
        for q in range(Q):
            for r in range(Rs):
                for warp in range(0, nthreads, 32):
                    addrs = []
                    for tid in range(warp, min(warp + 32, nthreads)):
                        g, j = thread(tid)
                        jj = j + q * TG; kk = jj & (Ns - 1)
                        base = ((jj // Ns) * Ns * Rs) + kk
                        addrs.append((g * (S if layout == 'col' else SM) + pad(base + r * Ns)) * E)
                    w_total += wavefronts(addrs, E); w_ideal += max(1, len(addrs) * E // 128)
        r_total = r_ideal = 0
        for k in range(R):
            for warp in range(0, nthreads, 32):
                addrs = []
                for tid in range(warp, min(warp + 32, nthreads)):
                    g, j = thread(tid)
                    addrs.append((g * (S if layout == 'col' else SM) + pad(j + TG * k)) * E)
                r_total += wavefronts(addrs, E); r_ideal += max(1, len(addrs) * E // 128)
        res.append((s, w_total / w_ideal, r_total / r_ideal))
    return res

if __name__ == '__main__':
    for E, LGRs in ((8, (3, 4, 5)), (16, (3, 4))):
        for LG in (8, 9, 10, 11, 12):
            for LGR in LGRs:
                L, R, TG, NP, lgR, radix = shape(LG, LGR)
                print(f"E={E} L={L} R={R} TG={TG} row:", [(s, round(w, 2), round(r, 2)) for s, w, r in simulate(LG, LGR, E, 'row')])
                for C in (2, 4, 8):
                    if C * TG > 1024: continue
                    best = min(range(0, 17), key=lambda cp: sum(w + r for _, w, r in simulate(LG, LGR, E, 'col', C, cp)))
                    print(f"      col C={C}: pad2", [(s, round(w, 2), round(r, 2)) for s, w, r in simulate(LG, LGR, E, 'col', C, 2)],
                          f"best pad {best}", [(s, round(w, 2), round(r, 2)) for s, w, r in simulate(LG, LGR, E, 'col', C, best)])
