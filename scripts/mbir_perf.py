"""MBIR per-iteration time at a config (default C5): hsnct_mbir with n and 0 iterations, CUDA
events on the launching stream; prints ms/iteration and the per-stage split from a 1-iteration
profile-free estimate (project / backproject / sqs timed by running hsnct_project and hsnct_fbp
is not the same launch configuration, so only the total is reported here; use ncu for the split)."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
import synthdata as sd  # noqa: E402
from paper_2410_22500_b200 import Hsnct  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
cfg = sd.CONFIGS[a.config]
h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
V = torch.rand((cfg.Np, cfg.K), generator=g, device=dev) * cfg.Nc
X0 = h.fbp(V).clamp_(min=0)
ws = h.workspace(5)
s = torch.cuda.current_stream()
res = {}
for n in (0, 1, a.iters):
    X = X0.clone()
    h.mbir(V, X, n, 5.0, 0.05, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    X = X0.clone()
    e0.record(s)
    h.mbir(V, X, n, 5.0, 0.05, ws=ws)
    e1.record(s)
    torch.cuda.synchronize()
    res[n] = e0.elapsed_time(e1)
h.sync()
per = (res[a.iters] - res[1]) / (a.iters - 1)
print(json.dumps({"config": cfg.name, "ms": res, "ms_per_iter": per, "setup_ms": res[1] - per}))
