"""Small end-to-end run of every kernel path for compute-sanitizer (memcheck / racecheck /
synccheck): decompose (persistent, per-iteration fallback, K > 8 two-pass), fbp, synthesize,
DHR, FMD on tiny shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_2410_22500_b200 import Hsnct  # noqa: E402

dev = torch.device("cuda:0")
for cfg, it in ((sd.custom(idx=40, Nc=24, Nv=10, Nr=2, Nk=70, K=3, M=3), 3),
                (sd.custom(idx=41, Nc=20, Nv=9, Nr=1, Nk=203, K=5, M=4), 2),
                (sd.custom(idx=42, Nc=16, Nv=8, Nr=1, Nk=40, K=10, M=5), 2)):
    pr = sd.make_problem(cfg, device=dev)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    V, D = pr["V0"].clone(), pr["D0"].clone()
    Ypad = torch.zeros((cfg.Np, (cfg.Nk + 3) // 4 * 4), device=dev)
    Ypad[:, :cfg.Nk] = pr["Y"]
    h.subspace_decompose(Ypad[:, :cfg.Nk], V, D, it, obj_trace=torch.zeros(2 * it, dtype=torch.float64, device=dev))
    X = h.fbp(V)
    h.synthesize(X, D, 0, cfg.Nr, 1, cfg.Nk - 2)
    h.dhr(Ypad[:, :cfg.Nk], 0, cfg.Nr, 0, cfg.Nk)
    nm = min(cfg.M, cfg.K, 8)
    lab = torch.as_tensor(sd.region_labels(pr), dtype=torch.int32).to(dev)
    lab[lab >= nm] = -1
    T = h.fmd_transform(X, lab.contiguous(), nm)
    h.fmd_materials(X, T)
    h.fmd_spectra(D, T)
    try:
        h.sync()
    except Exception as e:  # data errors (e.g. an empty region) are fine here
        print("deferred status:", e)
    h.close()
os.environ["HSNCT_NO_PERSIST"] = "1"
cfg = sd.custom(idx=43, Nc=20, Nv=9, Nr=1, Nk=64, K=4, M=3)
pr = sd.make_problem(cfg, device=dev)
h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
V, D = pr["V0"].clone(), pr["D0"].clone()
h.subspace_decompose(pr["Y"], V, D, 2)
h.sync()
torch.cuda.synchronize()
print("sanitize run ok")
