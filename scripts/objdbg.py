"""Objective trace of the GPU path vs the oracle for a few (K, N_k) shapes (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synthdata as sd  # noqa: E402
from paper_2410_22500_b200 import Hsnct  # noqa: E402

for K, M, Nk in ((6, 4, 801), (6, 4, 400), (7, 4, 300), (8, 4, 200), (6, 4, 80), (3, 3, 200)):
    c = sd.custom(idx=23, Nc=24, Nv=11, Nr=1, Nk=Nk, K=K, M=M)
    pr = sd.make_problem(c)
    h = Hsnct(c.Nv, c.Nr, c.Nc, c.Nk, c.K, device=0)
    n = 3
    ld = ((Nk + 3) // 4) * 4 + 4
    Yd = torch.zeros((c.Np, ld), device="cuda")
    Yd[:, :Nk] = pr["Y"].cuda()
    Yd = Yd[:, :Nk]
    V = pr["V0"].cuda().clone()
    D = pr["D0"].cuda().clone()
    obj = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
    h.subspace_decompose(Yd, V, D, n, obj_trace=obj)
    h.sync()
    Vo, Do, objo = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n, objective=True)
    ob = obj.cpu().numpy()
    print(K, M, Nk, os.environ.get("HSNCT_NO_PERSIST", ""), "max rel obj err %.2e" % np.max(np.abs(ob - objo) / objo),
          "V %.1e D %.1e" % (np.linalg.norm(V.cpu().numpy() - Vo) / np.linalg.norm(Vo),
                             np.linalg.norm(D.cpu().numpy() - Do) / np.linalg.norm(Do)))
