"""Per-iteration time of the FFMA persistent NMF kernel at C1 / C2 against the number of
persistent CTAs (HSNCT_NBLK caps the grid; the plan default is one CTA per SM).

  python scripts/nblk_sweep.py [configs=1,2] [n_iter=200] [nblk list=148,112,96,74,64,48,37,32,24,16]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2"]
n_iter = sys.argv[2] if len(sys.argv) > 2 else "200"
nbs = sys.argv[3].split(",") if len(sys.argv) > 3 else ["148", "112", "96", "74", "64", "48", "37", "32", "24", "16"]
for c in cfgs:
    for nb in nbs:
        env = dict(os.environ, HSNCT_NBLK=nb)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "tc_perf.py"), c, n_iter, "ffma"],
                           env=env, capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("C")]
        print(f"NBLK={nb}: " + (line[0] if line else ("FAILED " + r.stderr[-300:])), flush=True)
