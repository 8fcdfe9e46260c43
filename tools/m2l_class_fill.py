"""Fill factor of a class-batched M2L (CPU analysis with the oracle; not part of the product path).

M2L pairs (t, s) whose centre offset R = c_s - c_t is the same share one translation operator.
A CTA that owns a tile of T consecutive same-level targets and walks the distinct offset classes
of the tile does T x (#classes) row contractions; only the pairs are useful. This script counts
fill = pairs / (T x classes) for the BASELINE trees.

  python tools/m2l_class_fill.py C5 1048576
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402

CFG = {"C1": (1, 16384, 4, 64, 0.5), "C2": (2, 1 << 20, 6, 64, 0.5), "C3": (3, 1 << 20, 6, 64, 0.5),
       "C4": (4, 1 << 24, 8, 128, 0.4), "C5": (5, 1 << 22, 10, 64, 0.5)}


def main():
    name = sys.argv[1]
    cfg, n, p, ncrit, theta = CFG[name]
    if len(sys.argv) > 2:
        n = int(sys.argv[2])
    orc = oracle.Oracle()
    bodies = orc.generate_baseline_bodies(cfg, n, 1)
    t = orc.build_tree(bodies, ncrit, p)
    cells = t.cells()
    mo, ms, _, _ = orc.lists_csr(t, theta)
    nc = len(cells)
    cnt = np.diff(mo)
    tgt = np.repeat(np.arange(nc, dtype=np.int64), cnt)
    src = ms.astype(np.int64)
    npairs = len(src)
    lt, ls = cells.level[tgt].astype(np.int64), cells.level[src].astype(np.int64)
    print(f"{name} N={n}: cells {nc}, M2L pairs {npairs}, level diff histogram (s - t):",
          dict(zip(*np.unique(ls - lt, return_counts=True))))
    # offsets in units of half the smaller cell's half-side: radius = half-diagonal = h*sqrt(3)
    h = cells.radius
    hq = np.minimum(h[tgt], h[src]) * 0.5
    d = (cells.center[src] - cells.center[tgt]) / hq[:, None]
    k = np.rint(d).astype(np.int64)
    print("max |offset - integer|:", np.abs(d - k).max(), "offset range", k.min(), k.max())
    B = 256
    ckey = ((ls - lt + 2) * B + (k[:, 0] + B // 2)) * B * B + (k[:, 1] + B // 2) * B + (k[:, 2] + B // 2)
    assert (np.abs(k) < B // 2).all()
    print("distinct (level diff, offset) classes:", len(np.unique(ckey)),
          " with target level:", len(np.unique(ckey * 64 + lt)))
    # targets with lists, ordered by (level, index) = (level, Morton) since cells are level... check
    has = np.nonzero(cnt)[0]
    order = has[np.lexsort((cells.key[has], cells.level[has]))]
    for order_name, ordr in (("level,key", order), ("index", has)):
        rank = np.empty(nc, np.int64)
        rank[:] = -1
        rank[ordr] = np.arange(len(ordr))
        for T in (8, 16, 32, 64, 128):
            # tiles never straddle levels: rank within level
            lev = cells.level[ordr].astype(np.int64)
            first = np.zeros(len(ordr), np.int64)
            if order_name == "level,key":
                start = np.r_[0, np.nonzero(np.diff(lev))[0] + 1]
                first[start] = start
                first = np.maximum.accumulate(first)
                tile_of = (np.arange(len(ordr)) - first) // T + lev * (1 << 32)
            else:
                tile_of = np.arange(len(ordr)) // T
            tile_pair = tile_of[rank[tgt]]
            tk = np.unique(np.stack([tile_pair, ckey * 64 + lt], axis=1), axis=0)
            rows = len(tk) * T
            print(f"  order {order_name:9s} tile {T:4d}: tiles {len(np.unique(tile_of))}, tile-classes {len(tk)}, "
                  f"fill {npairs / rows:.3f}")


if __name__ == "__main__":
    main()
