"""Multi-rank sharding of the hot path (paper_2202_02870_b200/distributed.py) with gloo on the
CPU, world_size 2 and 3.  The per-shard arithmetic is injected (an engine built on the CPU
oracle — test infrastructure), so these tests check the row / slice blocking, both all-to-all
exchanges, the B-hat all-gather and the all-reduced stopping rule against the single-process
oracle on the same inputs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ltensor_oracle as O


class OracleEngine:
    """CPU engine with the device engine's interface (slice-major C-order stacks)."""

    def __init__(self, spec, trailing):
        self.spec = spec
        self.trailing = tuple(trailing)
        self.P = int(np.prod(trailing))

    @staticmethod
    def _into(res, out):
        if out is None:
            return res
        assert tuple(out.shape) == tuple(res.shape) and out.dtype == res.dtype
        out.copy_(res)
        return out

    def forward(self, x, out=None):
        a = x.numpy()
        h = O.forward(a, self.spec)
        res = torch.from_numpy(np.ascontiguousarray(h.reshape(a.shape[0], a.shape[1], self.P).transpose(2, 0, 1)))
        return self._into(res, out)

    def inverse(self, hat, real, out=None):
        h = hat.numpy()
        t = np.ascontiguousarray(h.transpose(1, 2, 0)).reshape((h.shape[1], h.shape[2]) + self.trailing)
        res = O.inverse(t, self.spec, assume_real=real)
        return self._into(torch.from_numpy(np.ascontiguousarray(res)), out)

    def slice_gemm(self, ah, bh, out=None):
        return self._into(torch.from_numpy(np.matmul(ah.numpy(), bh.numpy())), out)

    def svt(self, hat, tau):
        h = hat.numpy()
        if h.size == 0:
            return hat.clone()
        u, s, vh = np.linalg.svd(h, full_matrices=False)
        return torch.from_numpy(np.matmul(u * np.maximum(s - tau, 0.0)[:, None, :], vh))

    def gradient(self, xc, xp, pobs, mask, beta):
        y = xc + beta * (xc - xp)
        g = y - (torch.where(mask.bool(), y, torch.zeros_like(y)) - pobs)
        return y, g

    def norms(self, y, xn, gt):
        out = torch.zeros(4, dtype=torch.float64)
        out[0] = float(((y - xn).double() ** 2).sum())
        out[1] = float((xn.double() ** 2).sum())
        if gt is not None:
            out[2] = float(((xn - gt).double() ** 2).sum())
        out[3] = float(xn.max()) if xn.numel() else -np.inf
        return out


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as exc:  # surface worker failures immediately
        q.put((rank, exc))
        raise
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in procs:
        rank, val = q.get(timeout=120)
        if isinstance(val, Exception):
            for p in procs:
                p.kill()
            raise val
        results[rank] = val
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [results[r] for r in range(world)]


# ---- workers (module level so they pickle under spawn)
def _lproduct_worker(rank, world):
    from paper_2202_02870_b200.distributed import blocks, dist_l_product

    rng = np.random.default_rng(5)
    a = rng.standard_normal((7, 3, 2, 5))
    b = rng.standard_normal((3, 6, 2, 5))
    spec = O.ospec("dct", (7, 6, 2, 5))
    r0, r1 = blocks(7, world)[rank]
    k0, k1 = blocks(3, world)[rank]
    eng = OracleEngine(spec, (2, 5))
    c = dist_l_product(torch.from_numpy(a[r0:r1]), torch.from_numpy(b[k0:k1]), eng)
    ref = O.l_product(a, b, spec)[r0:r1]
    return float(np.abs(c.numpy() - ref).max())


def _svt_worker(rank, world):
    from paper_2202_02870_b200.distributed import blocks, dist_svt

    rng = np.random.default_rng(6)
    x = rng.standard_normal((9, 8, 3, 5))
    spec = O.ospec("fft", x.shape)
    r0, r1 = blocks(9, world)[rank]
    out = dist_svt(torch.from_numpy(x[r0:r1]), 0.8, 9, OracleEngine(spec, (3, 5)))
    ref = O.svt(x, 0.8, spec)[r0:r1]
    return float(np.abs(out.numpy() - ref).max())


def _pga_worker(rank, world):
    from paper_2202_02870_b200.completion import CompletionConfig
    from paper_2202_02870_b200.distributed import blocks, dist_pga_complete
    from paper_2202_02870_b200.transforms import make_spec

    rng = np.random.default_rng(7)
    spec_o = O.ospec("dct", (11, 9, 4))
    m = O.l_product(rng.standard_normal((11, 2, 4)), rng.standard_normal((2, 9, 4)), spec_o)
    mask = rng.random(m.shape) < 0.6
    r0, r1 = blocks(11, world)[rank]
    cfg = CompletionConfig(spec=make_spec("dct", m.shape), max_iters=25, tol=1e-3)
    x, trace = dist_pga_complete(torch.from_numpy(m[r0:r1]), torch.from_numpy(mask[r0:r1]), cfg, 11,
                                 OracleEngine(spec_o, (4,)), ground_truth_rows=torch.from_numpy(m[r0:r1]))
    ref, recs, status = O.pga_complete(m, mask, spec_o, max_iters=25, tol=1e-3, ground_truth=m)
    return (float(np.abs(x.numpy() - ref[r0:r1]).max()), trace.status == status, trace.iterations == len(recs),
            max((0.0 if r.rel_change == rr[3] else abs(r.rel_change - rr[3]) / max(rr[3], 1e-300))
                for r, rr in zip(trace.records, recs)),
            # mu0 = nu ||M||_F: the sharded sum differs from numpy's BLAS order in the last bits
            bool(np.allclose([r.mu for r in trace.records], [rr[1] for rr in recs], rtol=1e-14, atol=0)),
            max((0.0 if (np.isnan(r.rse) and np.isnan(rr[4])) else abs(r.rse - rr[4]) / rr[4])
                for r, rr in zip(trace.records, recs)))


def test_blocks_partition():
    from paper_2202_02870_b200.distributed import blocks

    for n in (0, 1, 7, 96, 300):
        for w in (1, 2, 3, 8):
            b = blocks(n, w)
            assert b[0][0] == 0 and b[-1][1] == n and all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1


@pytest.mark.parametrize("world", [2, 3])
def test_dist_l_product_gloo(world):
    assert max(run_ranks(_lproduct_worker, world)) < 1e-12


@pytest.mark.parametrize("world", [2, 3])
def test_dist_svt_gloo(world):
    assert max(run_ranks(_svt_worker, world)) < 1e-12


def test_dist_pga_gloo():
    for err, same_status, same_len, rel_err, mu_exact, rse_err in run_ranks(_pga_worker, 2):
        assert err < 1e-10 and same_status and same_len and mu_exact
        assert rel_err < 1e-9 and rse_err < 1e-9
