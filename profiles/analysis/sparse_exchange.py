"""How much would a sparse factor-row exchange (second half: "send only
the rows peers reference") save over the dense all-gather of the owned rows?

Host-only analysis on the synthetic configs (synth/, seeded): for G ranks with the whole-slice
partition of every mode (splatt_partition, C-14), rank q's local CSF for mode m holds the
nonzeros whose mode-m index is in q's range; the rows of A_n that q must hold for its MTTKRPs
of the other modes are the distinct mode-n indices of those nonzeros.  Dense exchange: q
receives every row it does not own.  Sparse exchange: q receives only referenced rows it does
not own.  Prints, per config / G / mode, the received-rows ratio sparse / dense (max over
ranks, which bounds the exchange time).

    python profiles/analysis/sparse_exchange.py [c2 c3 c5] > profiles/analysis/sparse_exchange.txt
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
import synth  # noqa: E402
import paper_1812_05961_b200 as sb  # noqa: E402  (host-only calls: no GPU needed)


def analyse(name, Gs=(2, 4, 8)):
    t = synth.generate_config(name)
    N, dims = len(t.dims), t.dims
    ind = [a.astype(np.int64) for a in t.ind]
    owner_of = []
    for G in Gs:
        bounds = [sb.partition(np.bincount(ind[m], minlength=dims[m]), G) for m in range(N)]
        # rank of each nonzero in each mode's partition
        rank_m = [np.searchsorted(bounds[m], ind[m], side="right") - 1 for m in range(N)]
        for n in range(N):
            dense, sparse = [], []
            for q in range(G):
                own = int(bounds[n][q + 1] - bounds[n][q])
                ref = np.zeros(dims[n], dtype=bool)
                for m in range(N):
                    if m != n:
                        ref[ind[n][rank_m[m] == q]] = True
                ref[bounds[n][q]:bounds[n][q + 1]] = False  # owned rows are local
                dense.append(dims[n] - own)
                sparse.append(int(ref.sum()))
            print(f"{name} G={G} mode {n} (I={dims[n]}): rows received per rank, max: dense "
                  f"{max(dense)}, sparse {max(sparse)}  ratio {max(sparse) / max(1, max(dense)):.3f}"
                  f"  (mean ratio {np.mean(sparse) / max(1, np.mean(dense)):.3f})", flush=True)
    del owner_of


if __name__ == "__main__":
    for c in sys.argv[1:] or ["c2", "c3", "c5"]:
        analyse(c)
