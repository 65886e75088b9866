"""GPU parity of the slice-sharded decomposition (NEXT-4; hsnct_nmf_begin / _rowpass / _dupdate,
paper_2410_22500_b200/sharded.py) against the fp64 oracle on the FULL problem.

* One rank on every row-pass plan (FFMA fused, tcgen05, two-pass K > 8): the split iteration
  computes what hsnct_subspace_decompose computes (V, D within 1e-5 of it, 1e-3 of the oracle,
  the objective trace within rtol 1e-3).
* Two ranks, each a process on this one GPU holding half of the slices, exchanging the
  per-iteration sums through gloo (the host does the exchange; no kernel waits on another
  rank's kernel): the concatenated V and the (identical) D match the oracle on all of Y.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synthdata as sd

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def rel(a, b):
    a = a.detach().cpu().double().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, np.float64)
    b = b.detach().cpu().double().numpy() if isinstance(b, torch.Tensor) else np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("plan,cfg,n_iter", [
    ("ffma", sd.custom(idx=81, Nc=24, Nv=10, Nr=4, Nk=200, K=4, M=3), 25),
    ("tc", sd.custom(idx=82, Nc=32, Nv=12, Nr=3, Nk=400, K=5, M=4), 20),
    ("mma", sd.custom(idx=84, Nc=32, Nv=12, Nr=3, Nk=400, K=5, M=4), 20),
    ("ffma", sd.custom(idx=83, Nc=20, Nv=9, Nr=2, Nk=96, K=10, M=4), 15),   # K > 8: two-pass
])
def test_sharded_one_rank_matches_decompose_and_oracle(monkeypatch, plan, cfg, n_iter):
    monkeypatch.setenv("HSNCT_NMF", plan)
    from paper_2410_22500_b200 import Hsnct
    from paper_2410_22500_b200.sharded import sharded_subspace_decompose
    pr = sd.make_problem(cfg)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    Y = pr["Y"].to(DEV)
    V, D = pr["V0"].to(DEV).clone(), pr["D0"].to(DEV).clone()
    obj = torch.zeros(2 * n_iter, dtype=torch.float64, device=DEV)
    sharded_subspace_decompose(h, Y, V, D, n_iter, obj_trace=obj)
    h.sync()
    V2, D2 = pr["V0"].to(DEV).clone(), pr["D0"].to(DEV).clone()
    h.subspace_decompose(Y, V2, D2, n_iter)
    h.sync()
    assert rel(V, V2) <= 1e-5 and rel(D, D2) <= 1e-5, (rel(V, V2), rel(D, D2))
    Vo, Do, objo = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n_iter, objective=True)
    assert rel(V, Vo) <= 1e-3 and rel(D, Do) <= 1e-3
    np.testing.assert_allclose(obj.cpu().numpy(), objo, rtol=1e-3)


def _rank(rank, world, port, cfg, n_iter, q):
    import torch.distributed as dist

    from paper_2410_22500_b200 import Hsnct
    from paper_2410_22500_b200.sharded import sharded_subspace_decompose, slice_range, slice_rows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        pr = sd.make_problem(cfg)
        r0, r1 = slice_range(cfg.Nr, rank, world)
        rows = slice_rows(cfg.Nv, cfg.Nr, cfg.Nc, r0, r1)
        h = Hsnct(cfg.Nv, r1 - r0, cfg.Nc, cfg.Nk, cfg.K, device=0)
        Y = pr["Y"][rows].to(DEV).contiguous()
        V = pr["V0"][rows].to(DEV).contiguous()
        D = pr["D0"].to(DEV).clone()
        obj = torch.zeros(2 * n_iter, dtype=torch.float64, device=DEV)
        sharded_subspace_decompose(h, Y, V, D, n_iter, obj_trace=obj)
        h.sync()
        q.put((rank, rows.numpy(), V.cpu().numpy(), D.cpu().numpy(), obj.cpu().numpy()))
        h.close()
    finally:
        dist.destroy_process_group()


def test_sharded_two_ranks_gloo_vs_oracle():
    cfg = sd.custom(idx=84, Nc=24, Nv=10, Nr=5, Nk=240, K=4, M=3)
    n_iter = 20
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, cfg, n_iter, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    pr = sd.make_problem(cfg)
    V = np.zeros((cfg.Np, cfg.K))
    for _, rows, Vr, _, _ in res:
        V[rows] = Vr
    assert np.array_equal(res[0][3], res[1][3]) and np.array_equal(res[0][4], res[1][4])  # replicated D, objective
    Vo, Do, objo = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n_iter, objective=True)
    assert rel(V, Vo) <= 1e-3 and rel(res[0][3], Do) <= 1e-3, (rel(V, Vo), rel(res[0][3], Do))
    np.testing.assert_allclose(res[0][4], objo, rtol=1e-3)
