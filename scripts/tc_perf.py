"""Row-pass throughput of the NMF plans on a config's shape (random Y+, values irrelevant to
speed): per-iteration time (CUDA events around n_iter iterations on the launching stream),
algorithmic GB/s = n_iter * (4 Np Nk + 8 Np K) / t, fraction of MEASURED_PEAKS hbm_gbs, and the
agreement of the plans' V, D after n_iter iterations from the same init.

  python scripts/tc_perf.py [config=5] [n_iter=10] [plans=tc,ffma]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthdata as sd  # noqa: E402


def main():
    ci = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    n_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    plans = sys.argv[3].split(",") if len(sys.argv) > 3 else ["tc", "ffma"]
    cfg = sd.CONFIGS[ci]
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    Y = torch.rand((cfg.Np, cfg.Nk), generator=g, device=dev) * 1.5 - 0.2
    V0 = torch.rand((cfg.Np, cfg.K), generator=g, device=dev) + 0.05
    D0 = torch.rand((cfg.K, cfg.Nk), generator=g, device=dev) + 0.05
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6461.5
    from paper_2410_22500_b200 import Hsnct
    res = {}
    for plan in plans:
        # "tcre": the tcgen05 pass with phase 2 re-streaming its chunks from L2
        # "mma16": K = 9..16 on the 16-warp form of the mma pass (default: 8 warps)
        os.environ["HSNCT_NMF"] = "tc" if plan.startswith("tc") else "mma" if plan.startswith("mma") else plan
        os.environ["HSNCT_MMA_MW"] = "16" if plan == "mma16" else "0"
        os.environ["HSNCT_TC_RESTREAM"] = "1" if plan == "tcre" else "0"
        h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
        V, D = V0.clone(), D0.clone()
        h.subspace_decompose(Y, V, D, 2)  # warm-up (and workspace allocation)
        h.sync()
        def timed(n):
            V, D = V0.clone(), D0.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            h.subspace_decompose(Y, V, D, n)
            e1.record()
            h.sync()
            return e0.elapsed_time(e1), V, D
        ms1, _, _ = timed(1)
        nh = max(1, n_iter // 2)
        msh, _, _ = timed(nh)
        ms, V, D = timed(n_iter)
        it_ms = (ms - msh) / max(1, n_iter - nh)  # marginal cost of one iteration (no input prep)
        by = n_iter * (4.0 * cfg.Np * cfg.Nk + 8.0 * cfg.Np * cfg.K)
        gbs = by / (ms * 1e-3) / 1e9
        gbi = (4.0 * cfg.Np * cfg.Nk + 8.0 * cfg.Np * cfg.K) / (it_ms * 1e-3) / 1e9
        print(f"C{ci} {h.debug_plan()}: {ms / n_iter:.3f} ms/iter incl. input prep (frac {gbs / peak:.3f}); "
              f"per iteration {it_ms:.4f} ms (frac {gbi / peak:.3f}); 1-iteration call {ms1:.3f} ms", flush=True)
        res[plan] = (V.cpu(), D.cpu())
        h.close()
        del h
        torch.cuda.empty_cache()
    if len(res) == 2:
        (Va, Da), (Vb, Db) = res.values()
        rv = float((Va.double() - Vb.double()).norm() / Vb.double().norm())
        rd = float((Da.double() - Db.double()).norm() / Db.double().norm())
        print(f"plans agree after {n_iter} it: V {rv:.2e} D {rd:.2e}")


if __name__ == "__main__":
    main()
