"""Registers / spills of the persistent NMF kernel instantiations for one K (ptxas -v).

  python scripts/regs.py 4 [LP NBG NGRP]
"""
import re
import subprocess
import sys

K = sys.argv[1] if len(sys.argv) > 1 else "4"
want = tuple(sys.argv[2:5])
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++20", "-lineinfo", "-Iinclude",
       "-Ipaper_2410_22500_b200/csrc", "-Xptxas", "-v", "-c", f"paper_2410_22500_b200/csrc/nmf_fused_k{K}.cu",
       "-o", f"/tmp/nmf_k{K}.o"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Function properties for \S*k_nmf_(persist|fused)ILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)E", line)
    if m:
        cur = (m.group(1),) + m.groups()[1:]
        continue
    if cur and "spill stores" in line:
        sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line).groups()
        cur = cur + sp
        continue
    if cur and "Used" in line and len(cur) == 7:
        r = re.search(r"Used (\d+) registers", line).group(1)
        if not want or cur[2:5] == want:
            print(f"{cur[0]:8s} K={cur[1]} LP={cur[2]} NBG={cur[3]} NG={cur[4]}  regs={r} spill st/ld={cur[5]}/{cur[6]}")
        cur = None
