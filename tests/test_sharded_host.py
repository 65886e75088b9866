"""Host logic of the slice-sharded decomposition (NEXT-4, paper_2410_22500_b200/sharded.py), on
CPU: the slice partition and row maps, and the per-iteration exchange under torch.distributed
with the gloo backend at world size 2 (a recording stand-in for the library handle: the
kernels themselves are covered by tests/test_gpu_sharded.py)."""
import os
import socket
import sys

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_22500_b200.sharded import slice_range, slice_rows, sharded_subspace_decompose  # noqa: E402


def test_slice_ranges_partition_and_balance():
    for Nr in (1, 2, 7, 64, 256):
        for world in (1, 2, 3, 8):
            if world > Nr:
                continue
            rs = [slice_range(Nr, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == Nr
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def test_slice_rows_are_the_slices_in_local_order():
    Nv, Nr, Nc = 5, 7, 3
    g = torch.arange(Nv * Nr * Nc).view(Nv, Nr, Nc)
    allrows = []
    for r0, r1 in ((0, 2), (2, 5), (5, 7)):
        rows = slice_rows(Nv, Nr, Nc, r0, r1)
        assert torch.equal(rows, g[:, r0:r1, :].reshape(-1))
        allrows.append(rows)
    assert torch.equal(torch.sort(torch.cat(allrows)).values, torch.arange(Nv * Nr * Nc))


class FakeHandle:
    """Records the call sequence; a rank's 'sums' are rank-dependent constants."""

    def __init__(self, rank, n):
        self.rank, self.n, self.calls, self.device = rank, n, [], torch.device("cpu")

    def nmf_red_size(self):
        return self.n

    def nmf_begin(self, Y, D, ws=None):
        self.calls.append(("begin",))

    def nmf_rowpass(self, Y, V, D, it, red, ws=None):
        red.copy_(torch.arange(self.n, dtype=torch.float64) * (self.rank + 1) + it)
        self.calls.append(("rowpass", it))

    def nmf_dupdate(self, D, red, it, obj2=None, ws=None):
        self.calls.append(("dupdate", it, red.clone()))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = FakeHandle(rank, 5)
        sharded_subspace_decompose(h, None, None, None, 3)
        q.put((rank, [(c[0],) + tuple(c[1:2]) for c in h.calls], [c[2].tolist() for c in h.calls if c[0] == "dupdate"]))
    finally:
        dist.destroy_process_group()


def test_exchange_gloo_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict((r, (calls, reds)) for r, calls, reds in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        calls, reds = res[r]
        assert calls == [("begin",)] + [x for it in range(3) for x in (("rowpass", it), ("dupdate", it))]
        for it, red in enumerate(reds):  # the all-reduced sums: sum over ranks of (i (rank+1) + it)
            assert red == [float(i * 3 + 2 * it) for i in range(5)]
