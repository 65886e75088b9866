"""Input preparation from uint8 counts (k_counts, NEXT-1) vs from fp32 Y (k_yplus) on a config's
shape: one-iteration decompositions from each input, CUDA events; random counts (Poisson)."""
import sys

import torch

sys.path.insert(0, ".")
import synthdata as sd  # noqa: E402
from paper_2410_22500_b200 import Hsnct  # noqa: E402

cfg = sd.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
y0 = torch.poisson(torch.full((cfg.Nr * cfg.Nc, cfg.Nk), cfg.counts, device=dev), generator=g).clamp(max=255).to(torch.uint8)
y = torch.poisson(torch.full((cfg.Np, cfg.Nk), 0.6 * cfg.counts, device=dev), generator=g).clamp(max=255).to(torch.uint8)
h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
Yb = torch.empty((cfg.Np, (cfg.Nk + 3) // 4 * 4), device=dev)
Y = h.counts_to_projections(y, y0, Y=Yb[:, :cfg.Nk])
V0 = torch.rand((cfg.Np, cfg.K), device=dev, generator=g) + 0.1
D0 = torch.rand((cfg.K, cfg.Nk), device=dev, generator=g) + 0.1
ws = h.workspace(7)
s = torch.cuda.current_stream()
for name, fn in (("fp32 Y", lambda V, D: h.subspace_decompose(Y, V, D, 1, ws=ws)),
                 ("counts", lambda V, D: h.subspace_decompose_counts(y, y0, V, D, 1, ws=ws))):
    ts = []
    for _ in range(3):
        V, D = V0.clone(), D0.clone()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn(V, D)
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{cfg.name} {name}: decompose(1 it) {min(ts):.3f} ms")
h.sync()
