"""Multi-GPU sharding of the *_L hot path, one process per GPU over
torch.distributed (NCCL on the B200s; gloo for the CPU tests).

Layout:
  * fibre phase (K1 / K1' / K4): rank g owns the i1-row block R_g of every tensor —
    tubes are independent under L, so the transforms need no communication;
  * slice phase (K3): rank h owns the contiguous slice block Q_h of the
    transform-domain stack;
  * the layout change between the two phases is one all-to-all each way: the
    forward transform's slice-major output is already destination-major (slice
    block Q_h is contiguous), so every send is contiguous;
  * l_product needs no all-to-all: A and C stay row-sharded, B is row-sharded
    over its l rows, transformed locally and all-gathered (B-hat is small);
  * PGA: the stopping-rule norms are partial sums per rank, one all-reduce per
    iteration (sums) plus one max (peak for psnr); the scalar recurrences run
    redundantly and identically on every rank.

The local compute is an `Engine`: `DeviceEngine` runs libltb on CUDA tensors of
the local shard; the CPU tests inject an engine built on the oracle to check
the sharding and the exchanges with gloo (tests/test_distributed.py).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from . import _native as nat
from .completion import CompletionConfig, CompletionTrace, IterationRecord, pga_schedule, rel_change
from .errors import ShapeError, UnsupportedSpecError
from .transforms import device_spec, forward_dtype

_TORCH_DT = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
             np.dtype(np.complex64): torch.complex64, np.dtype(np.complex128): torch.complex128}


def blocks(n: int, world: int) -> list:
    """Contiguous near-equal blocks [start, stop) of range(n) for `world` ranks."""
    base, extra = divmod(n, world)
    out, start = [], 0
    for r in range(world):
        stop = start + base + (1 if r < extra else 0)
        out.append((start, stop))
        start = stop
    return out


def _world(group):
    return dist.get_world_size(group), dist.get_rank(group)


# ----------------------------------------------------------------- device engine
def _view(t: torch.Tensor) -> nat.DeviceArray:
    dt = {torch.float32: np.float32, torch.float64: np.float64, torch.complex64: np.complex64,
          torch.complex128: np.complex128}[t.dtype]
    assert t.is_contiguous()
    return nat.DeviceArray(tuple(t.shape), dt, ptr=t.data_ptr(), owner=False)


class DeviceEngine:
    """libltb kernels on the CUDA tensors of this rank's shard (stream: torch's current)."""

    def __init__(self, spec, trailing):
        self.spec = spec
        self.trailing = tuple(int(d) for d in trailing)
        self.handle = device_spec(spec, self.trailing)
        self.P = self.handle.P
        # share torch's current stream (handle 0 = the legacy default stream, cudaStreamLegacy)
        s = torch.cuda.current_stream().cuda_stream
        nat.check(nat.lib().ltb_ctx_set_stream(nat.context(), s if s else 1))

    def _xform(self, x: torch.Tensor, rows: int, cols: int, inverse: bool, layout_in, layout_out, out_dtype):
        out_shape = (self.P, rows, cols) if layout_out == nat.SLICE_MAJOR else (rows, cols) + self.trailing
        out = torch.empty(out_shape, dtype=_TORCH_DT[np.dtype(out_dtype)], device=x.device)
        if out.numel():
            xv, ov = _view(x.contiguous()), _view(out)
            nat.check(nat.lib().ltb_transform(nat.context(), self.handle.ptr, rows * cols, int(inverse), xv.code,
                                              layout_in, xv.ptr, ov.code, layout_out, ov.ptr, None))
        return out

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """(rows, cols, trailing) -> slice-major (P, rows, cols)."""
        hat_dt = forward_dtype(np.dtype(str(x.dtype).replace("torch.", "")), self.spec)
        return self._xform(x, x.shape[0], x.shape[1], False, nat.TUBE_MAJOR, nat.SLICE_MAJOR, hat_dt)

    def inverse(self, hat: torch.Tensor, real: bool) -> torch.Tensor:
        dt = np.dtype(str(hat.dtype).replace("torch.", ""))
        out_dt = nat.real_of(dt) if real else dt
        return self._xform(hat, hat.shape[1], hat.shape[2], True, nat.SLICE_MAJOR, nat.TUBE_MAJOR, out_dt)

    def slice_gemm(self, ah: torch.Tensor, bh: torch.Tensor) -> torch.Tensor:
        P, m, k = ah.shape
        n = bh.shape[2]
        out = torch.empty((P, m, n), dtype=ah.dtype, device=ah.device)
        a, b, c = _view(ah.contiguous()), _view(bh.contiguous()), _view(out)
        nat.check(nat.lib().ltb_slice_gemm(nat.context(), a.code, P, m, n, k, nat.OP_N, a.ptr, k, m * k, nat.OP_N,
                                           b.ptr, n, k * n, c.ptr, n, m * n))
        return out

    def svt(self, hat: torch.Tensor, tau: float) -> torch.Tensor:
        out = torch.empty_like(hat)
        if hat.numel():
            h, o = _view(hat.contiguous()), _view(out)
            nat.check(nat.lib().ltb_slice_svt(nat.context(), h.code, hat.shape[0], hat.shape[1], hat.shape[2], h.ptr,
                                              float(tau), o.ptr))
        return out

    def gradient(self, xc, xp, pobs, mask_u8, beta):
        y, g = torch.empty_like(xc), torch.empty_like(xc)
        if xc.numel():
            nat.check(nat.lib().ltb_pga_gradient(nat.context(), _view(xc).code, xc.numel(), xc.data_ptr(),
                                                 xp.data_ptr(), pobs.data_ptr(), mask_u8.data_ptr(), float(beta),
                                                 y.data_ptr(), g.data_ptr()))
        return y, g

    def norms(self, y, xn, gt):
        """[sum (y - x+)^2, sum x+^2, sum (x+ - gt)^2, max x+] of the local shard (float64)."""
        import ctypes as C

        out = torch.zeros(4, dtype=torch.float64)
        if xn.numel():
            s = (C.c_double * 2)()
            v_xn, v_y = _view(xn), _view(y)
            nat.check(nat.lib().ltb_reduce_sumsq(nat.context(), v_y.code, xn.numel(), v_y.ptr, v_xn.ptr, s))
            out[0] = s[0]
            nat.check(nat.lib().ltb_reduce_sumsq(nat.context(), v_xn.code, xn.numel(), v_xn.ptr, None, s))
            out[1], out[3] = s[0], s[1]
            if gt is not None:
                v_gt = _view(gt)
                nat.check(nat.lib().ltb_reduce_sumsq(nat.context(), v_xn.code, xn.numel(), v_xn.ptr, v_gt.ptr, s))
                out[2] = s[0]
        else:
            out[3] = -math.inf
        return out


# ----------------------------------------------------------------- exchanges
def fibres_to_slices(hat_rows: torch.Tensor, I1: int, group=None) -> torch.Tensor:
    """(P, r_g, I2) on every rank g -> (|Q_h|, I1, I2) full slices of this rank's block Q_h."""
    world, rank = _world(group)
    P, r, I2 = hat_rows.shape
    qb = blocks(P, world)
    rb = blocks(I1, world)
    send = hat_rows.contiguous()
    in_splits = [(q1 - q0) * r * I2 for q0, q1 in qb]
    q0, q1 = qb[rank]
    out_splits = [(q1 - q0) * (r1 - r0) * I2 for r0, r1 in rb]
    recv = torch.empty(sum(out_splits), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send.reshape(-1), out_splits, in_splits, group=group)
    out = torch.empty((q1 - q0, I1, I2), dtype=send.dtype, device=send.device)
    off = 0
    for (r0, r1), n in zip(rb, out_splits):
        out[:, r0:r1, :] = recv[off:off + n].view(q1 - q0, r1 - r0, I2)
        off += n
    return out


def slices_to_fibres(slices: torch.Tensor, P: int, group=None) -> torch.Tensor:
    """(|Q_h|, I1, I2) on every rank h -> (P, r_g, I2) row block of this rank g (inverse exchange)."""
    world, rank = _world(group)
    nq, I1, I2 = slices.shape
    rb = blocks(I1, world)
    qb = blocks(P, world)
    send = torch.cat([slices[:, r0:r1, :].reshape(-1) for r0, r1 in rb]) if nq else slices.new_empty(0)
    in_splits = [nq * (r1 - r0) * I2 for r0, r1 in rb]
    r0, r1 = rb[rank]
    out_splits = [(b1 - b0) * (r1 - r0) * I2 for b0, b1 in qb]
    recv = torch.empty(sum(out_splits), dtype=slices.dtype, device=slices.device)
    dist.all_to_all_single(recv, send, out_splits, in_splits, group=group)
    return recv.view(P, r1 - r0, I2)


# ----------------------------------------------------------------- sharded operations
def dist_l_product(a_rows: torch.Tensor, b_rows: torch.Tensor, engine, group=None) -> torch.Tensor:
    """Row-sharded a *_L b (linalg.py:34-43): rank g holds rows R_g of A (I1 x l x ...) and the row
    block K_g of B (l x I2 x ...); returns rows R_g of C.  B-hat is all-gathered (NCCL all-gather);
    no all-to-all is needed."""
    world, _ = _world(group)
    ah = engine.forward(a_rows)                    # (P, r_g, l)
    bh_local = engine.forward(b_rows)              # (P, k_g, I2)
    sizes = [torch.zeros(1, dtype=torch.int64, device=bh_local.device) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([bh_local.shape[1]], dtype=torch.int64, device=bh_local.device), group=group)
    sizes = [int(s.item()) for s in sizes]
    kmax = max(sizes)
    P, _, I2 = bh_local.shape
    # all-gather needs equal blocks: pad the row block to the largest, trim after
    padded = bh_local.new_zeros((P, kmax, I2))
    padded[:, : bh_local.shape[1]] = bh_local
    parts = [bh_local.new_empty((P, kmax, I2)) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    bh = torch.cat([p[:, :s] for p, s in zip(parts, sizes)], dim=1)  # (P, l, I2)
    ch = engine.slice_gemm(ah, bh)
    real = not (a_rows.is_complex() or b_rows.is_complex())
    return engine.inverse(ch, real)


def dist_svt(x_rows: torch.Tensor, tau: float, I1: int, engine, group=None) -> torch.Tensor:
    """Row-sharded svt (linalg.py:168-181): transform rows, all-to-all to slice blocks, SVT,
    all-to-all back, inverse transform rows."""
    if tau < 0:
        from .errors import ParameterError

        raise ParameterError(f"tau must be >= 0, got {tau}")
    hat = engine.forward(x_rows)
    sl = fibres_to_slices(hat, I1, group)
    sl = engine.svt(sl, tau)
    back = slices_to_fibres(sl, hat.shape[0], group)
    return engine.inverse(back, not x_rows.is_complex())


def dist_pga_complete(m_rows: torch.Tensor, mask_rows: torch.Tensor, cfg: CompletionConfig, I1: int, engine,
                      group=None, ground_truth_rows=None, mu0=None):
    """Row-sharded pga_complete (completion.py:141-202).  Every rank returns its rows of the
    iterate and the (identical) trace.  `mu0` defaults to nu * ||M||_F over all ranks."""
    cfg.validate()
    if not cfg.spec.unitary_scaled:
        raise UnsupportedSpecError("completion uses SVT, which requires a unitary-scaled transform")
    if m_rows.shape != mask_rows.shape:
        raise ShapeError(f"mask shape {tuple(mask_rows.shape)} does not match data shape {tuple(m_rows.shape)}")
    mask_u8 = mask_rows.to(torch.uint8).contiguous()
    m_rows = m_rows.contiguous()
    pobs = torch.where(mask_rows.bool(), m_rows, torch.zeros_like(m_rows))

    def allsum(vals):
        t = torch.as_tensor(vals, dtype=torch.float64, device=m_rows.device)
        dist.all_reduce(t, group=group)
        return t

    if mu0 is None and cfg.mu0 is None:
        mu0 = cfg.nu * math.sqrt(float(allsum([float((m_rows.double() ** 2).sum())])[0]))
    elif mu0 is None:
        mu0 = float(cfg.mu0)
    mus, ts, betas = pga_schedule(cfg, mu0)
    pobs_zero = float(allsum([float((pobs.double() ** 2).sum())])[0]) == 0.0
    gt_sumsq = None
    if ground_truth_rows is not None and cfg.rse_denominator == "original":
        gt_sumsq = float(allsum([float((ground_truth_rows.double() ** 2).sum())])[0])
    x_prev = torch.zeros_like(m_rows)
    x_cur = torch.zeros_like(m_rows)
    trace = CompletionTrace()
    for k in range(1, cfg.max_iters + 1):
        y, g = engine.gradient(x_cur, x_prev, pobs, mask_u8, betas[k - 1])
        x_next = dist_svt(g, mus[k - 1], I1, engine, group)
        loc = engine.norms(y, x_next, ground_truth_rows)
        sums = allsum([float(loc[0]), float(loc[1]), float(loc[2])])
        peak = torch.tensor([float(loc[3])], dtype=torch.float64, device=m_rows.device)
        dist.all_reduce(peak, op=dist.ReduceOp.MAX, group=group)
        rel = rel_change(float(sums[0]), float(sums[1]), pobs_zero)
        rec = IterationRecord(k=k, mu=mus[k - 1], t=ts[k - 1], rel_change=rel)
        if ground_truth_rows is not None:
            den = math.sqrt(float(sums[1])) ** 2 if cfg.rse_denominator == "obtained" else gt_sumsq
            err = math.sqrt(float(sums[2])) ** 2
            rec.rse = math.nan if den == 0.0 else err / den
            pk = float(peak[0])
            rec.psnr = math.inf if err == 0.0 else (-math.inf if pk == 0.0 else 10.0 * math.log10(pk ** 2 / err))
        trace.records.append(rec)
        x_prev, x_cur = x_cur, x_next
        if rel <= cfg.tol:
            trace.status = "converged"
            break
    out = torch.where(mask_rows.bool(), m_rows, x_cur) if cfg.reimpose_observed else x_cur
    return out, trace
