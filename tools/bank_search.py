"""Shared-memory bank-conflict model for the sparse 3-D kernels' region tiles.

A warp-wide 8-byte shared load/store is served per half-warp: 16 lanes, 16 bank
pairs (one 8-byte slot each), so a half-warp costs max over slots of the number of
distinct elements mapping to the slot (element index mod 16).  This matched ncu's
shared wavefront counts on config 3 (162.5 M per interpolation launch predicted vs
measured).

  spread : k_spread3w cell-run flush -- lane (g0, g1, g2) = (lane >> 4,
           (lane >> 2) & 3, lane & 3) adds its 6 x 3 x 3 register tile at axis
           offsets (6 g0 + a, 3 g1 + b, 3 g2 + c).  Exhaustive search over axis
           orders and paddings (ak_q3w.cuh: Spread3wTile).
  interp : k_interp3m B-fragment loads (m8n8k4 column n = lane / 4, row kk = lane % 4;
           column pair i = 2 t + (n & 1) of quad n >> 1).  Axis orders and paddings.

Usage: python tools/bank_search.py [spread|interp]
"""
import itertools
import sys


def half_warp_wavefronts(elements):
    total = 0
    for h in range(2):
        slots = {}
        for el in elements[16 * h:16 * h + 16]:
            slots.setdefault(el % 16, set()).add(el)
        total += max(len(v) for v in slots.values())
    return total


def spread_cost(Sa, Sb, Sc):
    tot = 0
    for a, b, c in itertools.product(range(6), range(3), range(3)):
        els = [(6 * (l >> 4) + a) * Sa + (3 * ((l >> 2) & 3) + b) * Sb + (3 * (l & 3) + c) * Sc for l in range(32)]
        tot += half_warp_wavefronts(els)
    return tot


def interp_cost(Sa, Sb, Sc):
    tot = 0
    for t, ks in itertools.product(range(18), range(3)):
        els = []
        for l in range(32):
            n, kk = l >> 2, l & 3
            i = 2 * t + (n & 1)
            els.append((i // 3) * Sa + (3 * (n >> 1) + i % 3) * Sb + (4 * ks + kk) * Sc)
        tot += half_warp_wavefronts(els)
    return tot


def search(cost, pad=16):
    res = []
    for perm in itertools.permutations("abc"):
        for p1 in range(13, 13 + pad):
            for p2 in range(13 * p1, 13 * p1 + pad + 1):
                st = {perm[0]: 1, perm[1]: p1, perm[2]: p2}
                res.append((cost(st["a"], st["b"], st["c"]), 12 * (1 + p1 + p2) + 1, "".join(perm), p1, p2))
    res.sort(key=lambda r: (r[0], r[1]))
    return res


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "spread"
    cost = spread_cost if which == "spread" else interp_cost
    print("dense 13^3 (a, b, c) row-major:", cost(169, 13, 1), "wavefronts per 54 accesses; ideal 108")
    for r in search(cost)[:8]:
        print("cost %d  size %d  order (fastest first) %s  strides %d %d" % r)
