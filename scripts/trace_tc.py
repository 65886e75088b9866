"""Per-tile timeline of the tcgen05 row pass from its %globaltimer trace (TcStamp slots).

  python scripts/trace_tc.py [config=3]

Runs one decompose iteration (HSNCT_NMF=tc, HSNCT_TRACE=1) on random Y+ of the config's
shape and prints, averaged over tiles 8..255 of every CTA: the tile period, the epilogue's
wait for phase 1, its drain + exchange, the V update, the MMA thread's reaction to V and its
phase-2 issue time, and the producer's chunk-issue span (waits for free ring slots).
"""
import os
import sys

os.environ["HSNCT_TRACE"] = "1"
os.environ.setdefault("HSNCT_NMF", "tc")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_2410_22500_b200 import Hsnct  # noqa: E402

NAMES = ["EPI_START", "P1_SEEN", "X_SEEN", "V_READY", "P2_DRAINED", "MMA_P1_0", "MMA_P1_END", "MMA_P2_0",
         "MMA_P2_END", "LD_0", "LD_END", "V_DONE"]


def main():
    ci = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cfg = sd.CONFIGS[ci]
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    Y = torch.rand((cfg.Np, cfg.Nk), generator=g, device=dev)
    V = torch.rand((cfg.Np, cfg.K), generator=g, device=dev) + 0.05
    D = torch.rand((cfg.K, cfg.Nk), generator=g, device=dev) + 0.05
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    print(h.debug_plan())
    h.subspace_decompose(Y, V.clone(), D.clone(), 1)
    h.subspace_decompose(Y, V, D, 1)
    h.sync()
    tr = h.debug_trace().astype(np.int64)  # [tile, cta, 16]
    T = tr[8:256, :, :12].astype(np.float64)
    ok = (T > 0).all(axis=2)
    T = np.where(ok[..., None], T, np.nan)
    d = lambda a, b: np.nanmean(T[:, :, b] - T[:, :, a]) / 1e3  # noqa: E731  us
    per = np.nanmean(np.diff(T[:, :, 9], axis=0)) / 1e3
    print(f"tile period (producer LD_0 to LD_0)    {per:7.3f} us")
    print(f"producer: chunk copies of a tile        {d(9, 10):7.3f} us (LD_0 -> LD_END, waits for free slots)")
    print(f"MMA: LD_0 -> first chunk landed          {d(9, 5):7.3f} us")
    print(f"MMA: phase-1 issue (first chunk -> end) {d(5, 6):7.3f} us")
    print(f"epi: iteration start -> P1 complete     {d(0, 1):7.3f} us (waiting for phase 1)")
    print(f"epi: MMA P1 end -> P1 seen              {d(6, 1):7.3f} us")
    print(f"epi: P1 seen -> partials received       {d(1, 2):7.3f} us (drain + cluster exchange)")
    print(f"epi: received -> V computed             {d(2, 11):7.3f} us (sum, V update)")
    print(f"epi: V computed -> V ready              {d(11, 3):7.3f} us (operand writes, fence, barrier)")
    print(f"MMA: V ready -> phase 2 start           {d(3, 7):7.3f} us")
    print(f"MMA: phase-2 issue                      {d(7, 8):7.3f} us")
    print(f"epi: V ready -> phase 2 drained         {d(3, 4):7.3f} us")
    print(f"LD_0 -> V ready (tile latency)          {d(9, 3):7.3f} us")
    c0 = tr[8:14, 0, :12].astype(np.int64)
    base = c0[0, 9]
    print("cluster 0 rank 0, tiles 8..13 (us from tile 8 LD_0):")
    for i, row in enumerate(c0):
        print(f"  tile {8 + i}: " + " ".join(f"{n}={(v - base) / 1e3:.2f}" for n, v in zip(NAMES, row)))


if __name__ == "__main__":
    main()
