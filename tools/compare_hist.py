"""Compare per-cycle explicit relres of two big-run npz files (ours vs the
reference's): first cycle where they differ by more than given factors."""
import sys
import numpy as np


def cyc(f):
    d = np.load(f)
    e = d["h_expl"]
    it = d["h_iter"]
    m = ~np.isnan(e)
    return it[m], e[m], d


def main(a, b):
    ia, ea, da = cyc(a)
    ib, eb, db = cyc(b)
    k = min(len(ea), len(eb))
    rel = np.abs(np.log10(ea[:k]) - np.log10(eb[:k]))
    print(a, int(da["iters"]), "vs", b, int(db["iters"]), "cycles", len(ea), len(eb))
    for thr in (1e-12, 1e-9, 1e-6, 1e-3, 1e-2, 0.05, 0.3):
        bad = np.nonzero(rel > np.log10(1 + thr))[0]
        print("  first cycle with |rel diff| > %g: %s" % (thr, bad[0] if len(bad) else "none"))
    for c in (1, 5, 10, 20, 50, 100, 150, 200):
        if c < k:
            print("  cycle %3d iter %5d: %.6e vs %.6e" % (c, ia[c], ea[c], eb[c]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
