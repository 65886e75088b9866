"""FBP stage timings (ramp filter, backprojection) at a config's shape, random V, via
hsnct_debug_fbp_timing (CUDA events around each launch), median of 5; with the HBM and FP32
rooflines bench.py reports.

  python scripts/fbp_perf.py [config=5]
"""
import json
import math
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthdata as sd  # noqa: E402
from paper_2410_22500_b200 import Hsnct  # noqa: E402


def main():
    ci = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    cfg = sd.CONFIGS[ci]
    dev = torch.device("cuda:0")
    V = torch.rand((cfg.Np, cfg.K), device=dev)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    X = h.fbp(V)
    h.debug_fbp_timing(True)
    ts = []
    for _ in range(5):
        h.fbp(V, X)
        ts.append(h.debug_fbp_times())
    h.debug_fbp_timing(False)
    tr = statistics.median(t[0] for t in ts) * 1e-3
    tb = statistics.median(t[1] for t in ts) * 1e-3
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6461.5, "sm_max_mhz": 1965.0}
    K, Np, Nx = cfg.K, cfg.Np, cfg.Nx
    kc = K if K <= 8 else 16
    rb = 4.0 * K * Np + 4.0 * kc * Np
    P = 1 << max(1, (2 * cfg.Nc - 1).bit_length())
    flops = (cfg.Nv * cfg.Nr) * ((K + 1) // 2) * (2 * 5.0 * P * math.log2(P) + 2.0 * P)
    fp32 = 148 * 128 * 2 * peaks["sm_max_mhz"] * 1e6
    print(f"C{ci} ramp filter {tr * 1e3:.3f} ms: {rb / tr / 1e9:.0f} GB/s = {rb / tr / 1e9 / peaks['hbm_gbs']:.3f} of HBM, "
          f"FFT {flops / tr / 1e12:.1f} TFLOP/s = {flops / tr / fp32:.3f} of FP32")
    bp_fma = 2.0 * K * Nx * cfg.Nv
    print(f"C{ci} backprojection {tb * 1e3:.3f} ms: {bp_fma / tb / 1e12:.2f} T FMA/s = "
          f"{bp_fma / tb / (fp32 / 2):.3f} of the FP32 FMA peak")


if __name__ == "__main__":
    main()
