"""A plain-Python model of the exact in-order sum (csrc/b2o_xsum.cu), used by
the CPU suite to check the algorithm's arithmetic -- units per binade, the
tie parity rule, the two-variant run summaries and their merge, the
mirrored negative case -- against the definition (the sequential loop),
without a GPU.  Integers are Python ints (no overflow); the kernel's int32 /
int64 ranges are guarded by its own flags.  Formats: fp32 (MANT = 23) and
fp64 (MANT = 52), decoded from the IEEE bits with numpy."""

from __future__ import annotations

import math

import numpy as np

FMT = {np.float32: (23, 8, np.uint32), np.float64: (52, 11, np.uint64)}


def decode(x, dtype):
    """(sign, integer mantissa m, exponent ex) with |x| = m * 2^(ex - MANT)."""
    mant, ebits, ut = FMT[dtype]
    b = int(np.asarray(x, dtype).view(ut))
    neg = b >> (mant + ebits) & 1
    exr = b >> mant & ((1 << ebits) - 1)
    bias = (1 << (ebits - 1)) - 1
    m = b & ((1 << mant) - 1)
    if exr == (1 << ebits) - 1:
        return neg, None, None  # inf / nan
    if exr:
        return neg, m | (1 << mant), exr - bias
    return neg, m, 1 - bias


def units(x, e, dtype):
    """(c, tie) in units u = 2^(e - MANT): c = round(x/u) when not a tie,
    floor(x/u) for an exact half-way x (tie = 1); None when x can never stay
    in the binade (|x| >= 2^(e+1)) or is not finite."""
    neg, m, ex = decode(x, dtype)
    if m is None or ex - e > 0:
        return None
    d = ex - e
    if d == 0:
        c = m
        return (-c if neg else c), 0
    sh = -d
    q, rem, half = m >> sh, m & ((1 << sh) - 1), 1 << (sh - 1)
    if rem == half:
        return (-q - 1 if neg else q), 1
    c = q + (1 if rem > half else 0)
    return (-c if neg else c), 0


def summarise(xs, e, dtype):
    """Run summary for binade e: per start parity p, (P, lo, hi); None if a
    term is unusable."""
    out = []
    for p in (0, 1):
        P, lo, hi = 0, math.inf, -math.inf
        for x in xs:
            u = units(x, e, dtype)
            if u is None:
                return None
            c, tie = u
            r = c + (tie & ((p + P + c) & 1))
            P += r
            lo, hi = min(lo, P - 1), max(hi, P + 1)
        out.append((P, lo, hi))
    return out


def merge(a, b):
    """Run a then run b (both summaries for one binade)."""
    if a is None or b is None:
        return None
    out = []
    for p in (0, 1):
        Pa, la, ha = a[p]
        Pb, lb, hb = b[(p + Pa) & 1]
        out.append((Pa + Pb, min(la, Pa + lb), max(ha, Pa + hb)))
    return out


def apply(s, summ, dtype):
    """s after the run, or None when the summary is not usable from s."""
    mant = FMT[dtype][0]
    if summ is None or s == 0 or not np.isfinite(s):
        return None
    neg, m, ex = decode(s, dtype)
    if m < (1 << mant):  # subnormal
        return None
    P, lo, hi = summ[m & 1]
    if not neg:
        if m + lo < (1 << mant) or m + hi > (1 << (mant + 1)):
            return None
        m2 = m + P
    else:
        if m - hi < (1 << mant) or m - lo > (1 << (mant + 1)):
            return None
        m2 = m - P
    v = math.ldexp(m2, ex - mant)  # exact: m2 < 2^(MANT+1)
    return dtype(-v if neg else v)


def exact_sum(xs, s0, dtype, chunk=16, stats=None):
    """The model walk: apply each chunk's summary for the running sum's binade
    when usable, else add the chunk element by element (the definition)."""
    s = dtype(s0)
    stats = stats if stats is not None else {}
    stats.setdefault("fast", 0)
    stats.setdefault("slow", 0)
    for i in range(0, len(xs), chunk):
        part = xs[i:i + chunk]
        got = None
        if s != 0 and np.isfinite(s):
            e = decode(s, dtype)[2]
            got = apply(s, summarise(part, e, dtype), dtype)
        if got is None:
            stats["slow"] += 1
            for x in part:
                s = dtype(s + x)
        else:
            stats["fast"] += 1
            s = got
    return s
