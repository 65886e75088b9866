"""Phase breakdown of the persistent NMF kernel from its %globaltimer trace.

  HSNCT_TRACE=1 python scripts/trace_nmf.py [--config 2] [--n-iter 20]

Prints, averaged over iterations 2..n-1: the row pass (min / mean / max over CTAs),
the wait at grid barrier 1 (slowest CTA's pass end -> barrier passed), the D update,
barrier 2 + G + restage, and the whole iteration (wall, first start -> last end).
"""
import argparse
import os
import sys

os.environ.setdefault("HSNCT_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_2410_22500_b200 import Hsnct  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n-iter", type=int, default=20)
    a = ap.parse_args()
    cfg = sd.CONFIGS[a.config]
    dev = torch.device("cuda:0")
    pr = sd.make_problem(cfg, device=dev)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    for _ in range(2):
        V, D = pr["V0"].clone(), pr["D0"].clone()
        h.subspace_decompose(pr["Y"], V, D, a.n_iter)
        h.sync()
    tr = h.debug_trace()
    if tr is None:
        print("no trace (persistent path off?)")
        return
    n = min(a.n_iter, tr.shape[0])
    t = tr[:n].astype(np.int64)
    t = t - t[0, :, 0].min()
    us = 1e-3
    rows = []
    for it in range(2, n):
        s0, pe, b1, du, ie, pr, ds, gr = (t[it, :, j] for j in range(8))
        rows.append(dict(
            pass_min=(pe - s0).min() * us, pass_mean=(pe - s0).mean() * us, pass_max=(pe - s0).max() * us,
            bar1=(b1.max() - pe.max()) * us, dupd=(du - b1).mean() * us, dupd_max=(du - b1).max() * us,
            d_reduce=(pr - b1).mean() * us, d_update=(ds - pr).mean() * us, bar2=(gr.min() - du.max()) * us,
            g_restage=(gr - du).mean() * us, objective_tail=(ie - gr).mean() * us,
            bar2_restage=(ie - du).mean() * us, iter_wall=(ie.max() - s0.min()) * us,
            start_skew=(s0.max() - s0.min()) * us))
    keys = rows[0].keys()
    print(f"C{cfg.idx} K={cfg.K} Nk={cfg.Nk} Np={cfg.Np} n_iter={a.n_iter} CTAs={t.shape[1]}  (us, mean over iterations 2..{n - 1})")
    for k in keys:
        print(f"  {k:14s} {np.mean([r[k] for r in rows]):10.2f}")


if __name__ == "__main__":
    main()
