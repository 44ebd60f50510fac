"""Shared-memory bank-conflict model of the brick vmult kernel's passes (vmult_kernel.cuh), fp64 k=2,
brick 4x4x2: for every warp-wide access the number of wavefronts (64-bit: per half warp, max over the
16 bank pairs of the distinct words mapped to it). Used to choose pitches offline; see profiles/r02."""
import itertools
import sys

K, H = 2, 3
BX, BY, BZ = 4, 4, 2
NT = 256
S1 = S2 = S3 = 2


def odd(v):
    return v | 1


def B(a):
    return (BX, BY, BZ)[a]


def N(a):
    return B(a) * H


def O1(c):
    return 1 if c == 0 else 0


def O2(c):
    return 1 if c == 2 else 2


def LC(c):
    return N(c) + H + 1


def LO1H(c):
    return N(O1(c)) + 2 * H


def wavefronts(addrs):
    """64-bit accesses of one warp instruction (None = inactive lane)."""
    w = 0
    for half in (addrs[:16], addrs[16:]):
        act = [a for a in half if a is not None]
        if not act:
            continue
        per = {}
        for a in set(act):
            per.setdefault(a % 16, set()).add(a)
        w += max(len(v) for v in per.values())
    return w


def ideal(addrs):
    return sum(1 for half in (addrs[:16], addrs[16:]) if any(a is not None for a in half))


def run(c, UX, PCf, verbose=False):
    """returns (wavefronts, ideal) summed over the pass-1/2 accesses of component c"""
    PC = PCf(c)
    lc, lo1h = LC(c), LO1H(c)
    No1, No2 = N(O1(c)), N(O2(c))
    NO2, NO1 = B(O2(c)), B(O1(c))
    UY = LO1H(0) if c == 0 else (LC(1) if c == 1 else N(1) + 2 * H)
    US = UX if c == 2 else UX * UY
    tot = [0, 0]

    def acc(fn, n_items):
        # every thread loops it = tid, tid + NT, ...; warp w handles items w*32 .. w*32+31 of each round
        for base in range(0, n_items, 32):
            lanes = [base + l if base + l < n_items else None for l in range(32)]
            for addrs in fn(lanes):
                tot[0] += wavefronts(addrs)
                tot[1] += ideal(addrs)

    def ub(ci, oi):
        return oi * UX + ci if c == 0 else (ci * UX + oi if c == 1 else ci * UY * UX + oi)

    # pass 1 A1
    NLA = lc * lo1h

    def a1(lanes):
        out = []
        for j in range(S1 * H):
            ad = []
            for it in lanes:
                if it is None:
                    ad.append(None)
                    continue
                e2 = (it // NLA) * S1
                r = it % NLA
                ci = r % lc if c == 0 else r // lo1h
                oi = r // lc if c == 0 else r % lo1h
                ad.append(ub(ci, oi) + (e2 + 1) * H * US + j * US)
            out.append(ad)
        for a in range(S1 * H):
            ad = []
            for it in lanes:
                if it is None:
                    ad.append(None)
                    continue
                e2 = (it // NLA) * S1
                r = it % NLA
                ci = r % lc if c == 0 else r // lo1h
                oi = r // lc if c == 0 else r % lo1h
                ad.append(((e2 * H + a) * lo1h + oi) * PC + ci)
            out.append(ad)
        return out
    acc(a1, NLA * (NO2 // S1))
    NLB = lc * No1

    def b1(lanes):
        out = []
        for j in range((S1 + 2) * H):
            ad = []
            for it in lanes:
                if it is None:
                    ad.append(None)
                    continue
                e2 = (it // NLB) * S1
                r = it % NLB
                ci = r % lc if c == 0 else r // No1
                o = r // lc if c == 0 else r % No1
                ad.append(ub(ci, o + H) + e2 * H * US + j * US)
            out.append(ad)
        for a in range(S1 * H):
            ad = []
            for it in lanes:
                if it is None:
                    ad.append(None)
                    continue
                e2 = (it // NLB) * S1
                r = it % NLB
                ci = r % lc if c == 0 else r // No1
                o = r // lc if c == 0 else r % No1
                ad.append(((e2 * H + a) * No1 + o) * PC + ci)
            out.append(ad)
        return out
    acc(b1, NLB * (NO2 // S1))
    # pass 2
    NL = lc * No2

    def p2(lanes):
        out = []
        for j in range((S2 + 2) * H):
            ad = []
            for it in lanes:
                if it is None:
                    ad.append(None)
                    continue
                e1 = (it // NL) * S2
                r = it % NL
                ci, oj = r % lc, r // lc
                ad.append((oj * lo1h + e1 * H) * PC + ci + j * PC)
            out.append(ad)
        for j in range(S2 * H):
            for arr in (0, 1):
                ad = []
                for it in lanes:
                    if it is None:
                        ad.append(None)
                        continue
                    e1 = (it // NL) * S2
                    r = it % NL
                    ci, oj = r % lc, r // lc
                    ad.append((oj * No1 + e1 * H + j) * PC + ci)
                out.append(ad)
        return out
    acc(p2, NL * (NO1 // S2))
    # pass 3 reads
    NL3 = No1 * No2

    def p3(lanes):
        out = []
        for j in range((S3 + 1) * H + 1):
            ad = []
            for it in lanes:
                if it is None:
                    ad.append(None)
                    continue
                e0 = (it // NL3) * S3
                r = it % NL3
                oi, oj = r % No1, r // No1
                ad.append((oj * No1 + oi) * PC + e0 * H + j)
            out.append(ad)
        return out
    acc(p3, NL3 * (B(c) // S3))
    return tot


def main():
    base_ux = {0: 18, 1: 20, 2: 20}

    def pc_odd(c):
        return odd(LC(c))
    print("current (UX 18/20/20, PC = odd(LC)):")
    T = [0, 0]
    for c in range(3):
        t = run(c, base_ux[c], pc_odd)
        print("  C=%d wavefronts %d ideal %d (%.2fx)" % (c, t[0], t[1], t[0] / t[1]))
        T[0] += t[0]
        T[1] += t[1]
    print("  total %d ideal %d excess %.1f %%" % (T[0], T[1], 100 * (T[0] - T[1]) / T[0]))
    # search: UX for C=1,2 (even, >= 20) and PC per component (>= LC)
    best = None
    for ux1, ux2 in itertools.product(range(20, 52, 2), range(20, 52, 2)):
        for pcs in itertools.product(*[range(LC(c), LC(c) + 16) for c in range(3)]):
            tot = 0
            ok = True
            for c in range(3):
                t = run(c, (18, ux1, ux2)[c], lambda cc, p=pcs: p[cc])
                tot += t[0]
            if best is None or tot < best[0]:
                best = (tot, ux1, ux2, pcs)
        if ux2 == 20:
            print("progress", ux1, best, file=sys.stderr)
    print("best", best, "vs current", T[0], "ideal", T[1])


if __name__ == "__main__":
    main()


def run_padded(c, UX, PC, pad_a1, pad_b1):
    """pass 1 of component c with the o1 item extent padded to pad_a1 (A1) / pad_b1 (B1) lanes (C = 1, 2);
    returns (wavefronts, warp load/store instructions) of pass 1"""
    lc, lo1h = LC(c), LO1H(c)
    No1 = N(O1(c))
    NO2 = B(O2(c))
    UY = LC(1) if c == 1 else N(1) + 2 * H
    US = UX if c == 2 else UX * UY
    tot = [0, 0]

    def ub(ci, oi):
        return ci * UX + oi if c == 1 else ci * UY * UX + oi

    def acc(fn, n_items):
        for base in range(0, n_items, 32):
            lanes = [base + l if base + l < n_items else None for l in range(32)]
            for addrs in fn(lanes):
                if all(a is None for a in addrs):
                    continue
                tot[0] += wavefronts(addrs)
                tot[1] += 1

    P1 = pad_a1
    NLA = lc * P1

    def a1(lanes):
        out = []
        for j in range(2 * S1 * H):
            ad = []
            for it in lanes:
                if it is None:
                    ad.append(None)
                    continue
                e2 = (it // NLA) * S1
                r = it % NLA
                ci, oi = r // P1, r % P1
                if oi >= lo1h:
                    ad.append(None)
                    continue
                if j < S1 * H:
                    ad.append(ub(ci, oi) + (e2 + 1) * H * US + j * US)
                else:
                    ad.append(((e2 * H + j - S1 * H) * lo1h + oi) * PC + ci)
            out.append(ad)
        return out
    acc(a1, NLA * (NO2 // S1))
    P2 = pad_b1
    NLB = lc * P2

    def b1(lanes):
        out = []
        for j in range((S1 + 2) * H + S1 * H):
            ad = []
            for it in lanes:
                if it is None:
                    ad.append(None)
                    continue
                e2 = (it // NLB) * S1
                r = it % NLB
                ci, o = r // P2, r % P2
                if o >= No1:
                    ad.append(None)
                    continue
                if j < (S1 + 2) * H:
                    ad.append(ub(ci, o + H) + e2 * H * US + j * US)
                else:
                    ad.append(((e2 * H + j - (S1 + 2) * H) * No1 + o) * PC + ci)
            out.append(ad)
        return out
    acc(b1, NLB * (NO2 // S1))
    return tot
