#!/usr/bin/env python
"""Shared-memory bank check of the slab-ring interpolation kernel's B-fragment
reads (spread_interp.cu: k_interp_push_slab), used to pick the column stride CS
and the slab padding.

Lane l of a warp (g = l >> 2, t = l & 3) reads, for k-step ks and n-tile nt,
the double at
    slot(V + zl // SBZ) * SLAB + ((cy + oy) * CS + cx + ox) * 3 * SBZ + zl % SBZ (+ d SBZ)
with zl = 8 nt + g, (cx, cy) = divmod-position of column 4 ks + t in the
m-tile's window of width RXm, (ox, oy) the window origin in the brick tile.
A 64-bit warp load is served in 2 wavefronts (half-warps) when the 16 lanes of
each half hit 16 distinct 8-byte bank slots; the script reports the worst and
the mean number of wavefronts per half-warp over every window shape, origin,
ring slot and k-step.

  python tools/slab_banks.py
"""


def check(w, ib, m, sbz, cs, slab, ns, rz):
    worst, tot, cnt = 0, 0, 0
    for ex in range(ib):
        for ey in range(ib):
            rxm, rym = w + ex, w + ey
            ks_n = (rxm * rym + 3) // 4
            for ox in range(0, (m - 1) * ib + ib - ex):
                for oy in (0, (m - 1) * ib + ib - 1 - ey):
                    for v in range(ns):
                        for nt in range(rz // 8):
                            for ks in range(ks_n):
                                for h in (0, 1):
                                    slots = {}
                                    for g in range(4 * h, 4 * h + 4):
                                        zl = 8 * nt + g
                                        base = ((v + zl // sbz) % ns) * slab + zl % sbz
                                        for t in range(4):
                                            c = 4 * ks + t
                                            cx, cy = c % rxm, c // rxm
                                            a = base + ((cy + oy) * cs + cx + ox) * 3 * sbz
                                            slots.setdefault(a % 16, set()).add(a // 16)
                                    way = max(len(s) for s in slots.values())
                                    worst = max(worst, way)
                                    tot += way
                                    cnt += 1
    return worst, tot / cnt


def main():
    # (name, w, ib, m, SBZ, CS, rows per slab, ring NS, RZ)
    cases = [("w=13, CS 18, zero row", 13, 2, 2, 4, 18, 17, 5, 16),
             ("w=13, CS 17, no zero row", 13, 2, 2, 4, 17, 16, 6, 16),
             ("w=8 dense, CS 17", 8, 3, 3, 1, 17, 17, 12, 8),
             ("w=5 dense, CS 9", 5, 2, 2, 4, 9, 9, 4, 8)]
    for name, w, ib, m, sbz, cs, rows, ns, rz in cases:
        slab = rows * cs * 3 * sbz
        if sbz == 1:
            slab += (20 - slab % 16) % 16  # one-row slabs padded to 4 (mod 16)
        worst, mean = check(w, ib, m, sbz, cs, slab, ns, rz)
        print(f"{name:28s} slab {slab:5d} doubles: worst {worst}-way, mean {mean:.3f} wavefronts/half-warp")


if __name__ == "__main__":
    main()
