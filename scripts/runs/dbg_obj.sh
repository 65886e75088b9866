HSNCT_LIB=$PWD/paper_2410_22500_b200/libhsnct_dbg.so python - <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import torch, synthdata as sd
from paper_2410_22500_b200 import Hsnct
c = sd.custom(idx=23, Nc=24, Nv=11, Nr=1, Nk=801, K=6, M=4); pr = sd.make_problem(c)
h = Hsnct(c.Nv, c.Nr, c.Nc, c.Nk, c.K, device=0)
Yd = torch.zeros((c.Np, 808), device="cuda"); Yd[:, :801] = pr["Y"].cuda(); Yd = Yd[:, :801]
V = pr["V0"].cuda().clone(); D = pr["D0"].cuda().clone()
obj = torch.zeros(2, dtype=torch.float64, device="cuda")
h.subspace_decompose(Yd, V, D, 1, obj_trace=obj); h.sync(); torch.cuda.synchronize()
print(obj.cpu().numpy())
PY
