"""Per-call timing of the FMD back half at a BASELINE config (diagnostics).

  python scripts/time_fmd.py [--config 4] [--n-iter 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_2410_22500_b200 import Hsnct  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n-iter", type=int, default=2)
    a = ap.parse_args()
    cfg = sd.CONFIGS[a.config]
    dev = torch.device("cuda:0")
    pr = sd.make_problem(cfg, device=dev)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    V, D = pr["V0"].clone(), pr["D0"].clone()
    h.subspace_decompose(pr["Y"], V, D, a.n_iter)
    X = h.fbp(V)
    nm = min(cfg.M, cfg.K)
    lab = torch.as_tensor(sd.region_labels(pr), dtype=torch.int32).to(dev).contiguous()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for rep in range(3):
        e = [ev() for _ in range(4)]
        e[0].record()
        T = h.fmd_transform(X, lab, nm)
        e[1].record()
        Xm = h.fmd_materials(X, T)
        e[2].record()
        Dm = h.fmd_spectra(D, T)
        e[3].record()
        torch.cuda.synchronize()
        print(f"rep {rep}: transform {e[0].elapsed_time(e[1]):.3f} ms, materials {e[1].elapsed_time(e[2]):.3f} ms, "
              f"spectra {e[2].elapsed_time(e[3]):.3f} ms")
        del Xm, Dm


if __name__ == "__main__":
    main()
