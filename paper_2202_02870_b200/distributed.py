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

    def _xform(self, x: torch.Tensor, rows: int, cols: int, inverse: bool, layout_in, layout_out, out_dtype,
               out=None):
        out_shape = (self.P, rows, cols) if layout_out == nat.SLICE_MAJOR else (rows, cols) + self.trailing
        if out is None:
            out = torch.empty(out_shape, dtype=_TORCH_DT[np.dtype(out_dtype)], device=x.device)
        elif tuple(out.shape) != out_shape or out.dtype != _TORCH_DT[np.dtype(out_dtype)] or not out.is_contiguous():
            raise ShapeError(f"out must be a contiguous {out_shape} {np.dtype(out_dtype)} tensor")
        if out.numel():
            xv, ov = _view(x.contiguous()), _view(out)
            nat.check(nat.lib().ltb_transform(nat.context(), self.handle.ptr, rows * cols, int(inverse), xv.code,
                                              layout_in, xv.ptr, ov.code, layout_out, ov.ptr, None))
        return out

    def forward(self, x: torch.Tensor, out=None) -> torch.Tensor:
        """(rows, cols, trailing) -> slice-major (P, rows, cols)."""
        hat_dt = forward_dtype(np.dtype(str(x.dtype).replace("torch.", "")), self.spec)
        return self._xform(x, x.shape[0], x.shape[1], False, nat.TUBE_MAJOR, nat.SLICE_MAJOR, hat_dt, out)

    def inverse(self, hat: torch.Tensor, real: bool, out=None) -> torch.Tensor:
        dt = np.dtype(str(hat.dtype).replace("torch.", ""))
        out_dt = nat.real_of(dt) if real else dt
        return self._xform(hat, hat.shape[1], hat.shape[2], True, nat.SLICE_MAJOR, nat.TUBE_MAJOR, out_dt, out)

    def slice_gemm(self, ah: torch.Tensor, bh: torch.Tensor, out=None) -> torch.Tensor:
        P, m, k = ah.shape
        n = bh.shape[2]
        if out is None:
            out = torch.empty((P, m, n), dtype=ah.dtype, device=ah.device)
        elif tuple(out.shape) != (P, m, n) or out.dtype != ah.dtype or not out.is_contiguous():
            raise ShapeError(f"out must be a contiguous {(P, m, n)} {ah.dtype} tensor")
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

    def svt_carried(self, hat: torch.Tensor, tau: float, state: dict) -> torch.Tensor:
        """svt of this rank's slices warm-started from the right bases of the previous call
        (ltb_slice_svt_carry, the fp32 PGA path of ltb_pga_run); `state` keeps the bases
        between iterations.  Other dtypes and slices narrower than 32 use ltb_slice_svt."""
        nb, m, n = hat.shape
        if hat.dtype != torch.float32 or min(m, n) < 32 or not hat.numel():
            return self.svt(hat, tau)
        if state.get("v") is None or state["v"].shape[0] != nb:
            state["v"] = torch.empty((nb, min(m, n), min(m, n)), dtype=torch.float32, device=hat.device)
            state["warm"] = 0
        out = torch.empty_like(hat)
        h = hat.contiguous()
        nat.check(nat.lib().ltb_slice_svt_carry(nat.context(), nb, m, n, h.data_ptr(), float(tau), out.data_ptr(),
                                                state["v"].data_ptr(), int(state["warm"])))
        state["warm"] = 1
        return out

    def norms_device(self, y, xn, gt) -> torch.Tensor:
        """As `norms`, left on the device (float64 [sum (y - x+)^2, sum x+^2, sum (x+ - gt)^2,
        max x+]) with no host synchronisation."""
        buf = torch.zeros(6, dtype=torch.float64, device=xn.device)
        if xn.numel():
            lib, ctx, code = nat.lib(), nat.context(), _view(xn).code
            nat.check(lib.ltb_reduce_sumsq_device(ctx, code, xn.numel(), y.data_ptr(), xn.data_ptr(), buf.data_ptr()))
            nat.check(lib.ltb_reduce_sumsq_device(ctx, code, xn.numel(), xn.data_ptr(), None, buf[2:].data_ptr()))
            if gt is not None:
                nat.check(lib.ltb_reduce_sumsq_device(ctx, code, xn.numel(), xn.data_ptr(), gt.data_ptr(),
                                                      buf[4:].data_ptr()))
        else:
            buf[3] = -math.inf
        return torch.stack([buf[0], buf[2], buf[4], buf[3]])

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
    if I1 % world == 0:  # equal row blocks: the reassembly is one permuting copy
        return recv.view(world, q1 - q0, I1 // world, I2).transpose(0, 1).reshape(q1 - q0, I1, I2)
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
    if not nq:
        send = slices.new_empty(0)
    elif I1 % world == 0:  # equal row blocks: destination-major in one permuting copy
        send = slices.view(nq, world, I1 // world, I2).transpose(0, 1).reshape(-1)
    else:
        send = torch.cat([slices[:, r0:r1, :].reshape(-1) for r0, r1 in rb])
    in_splits = [nq * (r1 - r0) * I2 for r0, r1 in rb]
    r0, r1 = rb[rank]
    out_splits = [(b1 - b0) * (r1 - r0) * I2 for b0, b1 in qb]
    recv = torch.empty(sum(out_splits), dtype=slices.dtype, device=slices.device)
    dist.all_to_all_single(recv, send, out_splits, in_splits, group=group)
    return recv.view(P, r1 - r0, I2)


# ----------------------------------------------------------------- sharded operations
class DistLProductPlan:
    """Row-sharded a *_L b (linalg.py:34-43) with every buffer allocated once.

    Rank g holds rows R_g of A (r_g x l x trailing) and the row block K_g of B (k_g x I2 x
    trailing) and produces rows R_g of C.  One step: K1 of both local operands into
    slice-major buffers, an all-gather of the B-hat row blocks straight into one contiguous
    (world, P, kmax, I2) buffer (the only exchange; no all-to-all is needed), one permute to
    (P, l, I2), the slice GEMM and K1'.  The row-block sizes are exchanged once here (the
    only host synchronisation), so `run` is a fixed launch sequence on the current stream."""

    def __init__(self, a_shape, b_shape, engine, dtype: torch.dtype, device, group=None, exchange=None):
        self.engine, self.group = engine, group
        self.world, self.rank = _world(group)
        # exchange=True keeps the all-gather + permute even on one rank (tests of that path)
        self.exchange = self.world > 1 if exchange is None else bool(exchange)
        a_shape, b_shape = tuple(a_shape), tuple(b_shape)
        r, l = a_shape[:2]
        k_g, I2 = b_shape[:2]
        if a_shape[2:] != b_shape[2:] or a_shape[2:] != tuple(engine.trailing):
            raise ShapeError(f"trailing dims of {a_shape} and {b_shape} must both be {tuple(engine.trailing)}")
        sizes = torch.zeros(self.world, dtype=torch.int64, device=device)
        mine = torch.tensor([k_g], dtype=torch.int64, device=device)
        if self.world > 1:
            dist.all_gather_into_tensor(sizes, mine, group=group)
        else:
            sizes.copy_(mine)
        self.sizes = [int(v) for v in sizes.tolist()]
        if sum(self.sizes) != l:
            raise ShapeError(f"B row blocks {self.sizes} do not add up to A's column count {l}")
        np_dt = np.dtype(str(dtype).replace("torch.", ""))
        hat_t = _TORCH_DT[np.dtype(forward_dtype(np_dt, engine.spec))]
        P, kmax = engine.P, max(self.sizes)
        self.a_shape, self.b_shape, self.dtype = a_shape, b_shape, dtype
        self.real = not dtype.is_complex
        self.k_g, self.kmax, self.I2, self.l, self.P = k_g, kmax, I2, l, P
        new = lambda *shape, dt=hat_t: torch.empty(shape, dtype=dt, device=device)
        self.ha = new(P, r, l)
        self.hc = new(P, r, I2)
        # own row block, padded to kmax rows so every rank contributes an equal all-gather block
        self.hb_loc = torch.zeros((P, kmax, I2), dtype=hat_t, device=device)
        self.hb_tmp = None if k_g == kmax else new(P, k_g, I2)
        self.equal = len(set(self.sizes)) == 1
        if not self.exchange:
            self.hb_all, self.hb, self.rows = None, self.hb_loc, None
        else:
            self.hb_all = new(self.world * P * kmax * I2)
            self.hb = new(P, l, I2)
            # unequal blocks: the valid rows of the permuted (P, world * kmax, I2) gather
            self.rows = None if self.equal else torch.tensor(
                [g * kmax + i for g, s in enumerate(self.sizes) for i in range(s)], dtype=torch.int64, device=device)
        self.c_shape = (r, I2) + tuple(engine.trailing)

    def _check(self, a, b):
        if tuple(a.shape) != self.a_shape or tuple(b.shape) != self.b_shape:
            raise ShapeError(f"plan was built for A {self.a_shape}, B {self.b_shape}; got {tuple(a.shape)}, "
                             f"{tuple(b.shape)}")

    def _local(self, a, b):
        """Phase 1: K1 of the local A rows and B row block (no communication)."""
        eng = self.engine
        eng.forward(a, out=self.ha)
        if self.hb_tmp is None:
            eng.forward(b, out=self.hb_loc)
        else:
            eng.forward(b, out=self.hb_tmp)
            self.hb_loc[:, : self.k_g].copy_(self.hb_tmp)

    def _exchange(self):
        """Phase 2: the B-hat all-gather (the only collective)."""
        if self.exchange:
            dist.all_gather_into_tensor(self.hb_all, self.hb_loc.reshape(-1), group=self.group)

    def _finish(self, out):
        """Phase 3: permute the gathered blocks to (P, l, I2), slice GEMM, K1'."""
        if self.exchange:
            P, W, kmax, I2 = self.P, self.world, self.kmax, self.I2
            gathered = self.hb_all.view(W, P, kmax, I2).transpose(0, 1)  # (P, W, kmax, I2)
            if self.equal:
                self.hb.view(P, W, kmax, I2).copy_(gathered)
            else:
                torch.index_select(gathered.reshape(P, W * kmax, I2), 1, self.rows, out=self.hb)
        self.engine.slice_gemm(self.ha, self.hb, out=self.hc)
        return self.engine.inverse(self.hc, self.real, out=out)

    def run(self, a: torch.Tensor, b: torch.Tensor, out=None) -> torch.Tensor:
        self._check(a, b)
        self._local(a, b)
        self._exchange()
        return self._finish(out)

    def graphed(self, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, stream):
        """Capture the two compute phases for the fixed buffers a, b, out as CUDA graphs on
        `stream` (the stream the engine's context launches on) and return a step callable:
        replay phase 1, the all-gather eagerly on the same stream, replay phase 3.  The
        collective stays outside the graphs so capture never depends on the NCCL build."""
        self._check(a, b)
        self.run(a, b, out=out)  # settle kernel attributes / tensor-map caches before capture
        g1, g3 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        if not self.exchange:
            with torch.cuda.graph(g3, stream=stream):  # no collective: one graph for the whole step
                self._local(a, b)
                self._finish(out)
            return g3.replay
        with torch.cuda.graph(g1, stream=stream):
            self._local(a, b)
        with torch.cuda.graph(g3, stream=stream):
            self._finish(out)

        def step():
            g1.replay()
            self._exchange()
            g3.replay()

        return step


def dist_l_product(a_rows: torch.Tensor, b_rows: torch.Tensor, engine, group=None, out=None) -> torch.Tensor:
    """Row-sharded a *_L b (linalg.py:34-43): rank g holds rows R_g of A (I1 x l x ...) and the row
    block K_g of B (l x I2 x ...); returns rows R_g of C.  B-hat is all-gathered (NCCL all-gather);
    no all-to-all is needed.  The DistLProductPlan is cached on the engine per shape/dtype."""
    key = (tuple(a_rows.shape), tuple(b_rows.shape), a_rows.dtype, str(a_rows.device), id(group))
    plans = engine.__dict__.setdefault("_dist_plans", {})
    plan = plans.get(key)
    if plan is None:
        if a_rows.dtype != b_rows.dtype:
            raise ShapeError(f"operand dtypes differ: {a_rows.dtype} vs {b_rows.dtype}")
        plan = plans[key] = DistLProductPlan(a_rows.shape, b_rows.shape, engine, a_rows.dtype, a_rows.device, group)
    return plan.run(a_rows.contiguous(), b_rows.contiguous(), out=out)


def dist_svt(x_rows: torch.Tensor, tau: float, I1: int, engine, group=None, carry=None) -> torch.Tensor:
    """Row-sharded svt (linalg.py:168-181): transform rows, all-to-all to slice blocks, SVT,
    all-to-all back, inverse transform rows.  `carry` (a dict kept by the caller across PGA
    iterations) selects the engine's warm-started SVT when it has one."""
    if tau < 0:
        from .errors import ParameterError

        raise ParameterError(f"tau must be >= 0, got {tau}")
    hat = engine.forward(x_rows)
    sl = fibres_to_slices(hat, I1, group)
    if carry is not None and hasattr(engine, "svt_carried"):
        sl = engine.svt_carried(sl, tau, carry)
    else:
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
    if isinstance(engine, DeviceEngine) and m_rows.is_cuda:
        return _dist_pga_device(m_rows, mask_rows, cfg, I1, engine, group, ground_truth_rows, mu0)
    mask_u8 = mask_rows.to(torch.uint8).contiguous()
    m_rows = m_rows.contiguous()
    pobs = torch.where(mask_u8.bool(), m_rows, torch.zeros_like(m_rows)).contiguous()

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
    carry = {}  # right singular bases of this rank's slices, carried between iterations
    on_device = hasattr(engine, "norms_device")
    for k in range(1, cfg.max_iters + 1):
        y, g = engine.gradient(x_cur, x_prev, pobs, mask_u8, betas[k - 1])
        x_next = dist_svt(g, mus[k - 1], I1, engine, group, carry=carry)
        if on_device:  # reduce on the device; one host synchronisation per iteration
            loc = engine.norms_device(y, x_next, ground_truth_rows)
            sums, peak = loc[:3].clone(), loc[3:].clone()
            dist.all_reduce(sums, group=group)
            dist.all_reduce(peak, op=dist.ReduceOp.MAX, group=group)
            both = torch.cat([sums, peak]).tolist()
            sums, peak = both[:3], both[3:]
        else:
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
    out = torch.where(mask_u8.bool(), m_rows, x_cur).contiguous() if cfg.reimpose_observed else x_cur
    return out, trace


def _dist_pga_device(m_rows, mask_rows, cfg, I1, engine, group, gt_rows, mu0, chunk: int = 16):
    """The device path of dist_pga_complete: per iteration one fused gradient + forward launch
    (ltb_pga_shard_forward), the fibre -> slice all-to-all, the slice block's SVT warm-started
    from the previous iteration's right bases (ltb_pga_shard_svt), the all-to-all back, one
    fused inverse + norms launch (ltb_pga_shard_inverse), two all-reduces of the five sums and
    the stop decision on the device (ltb_pga_shard_decide).  Nothing synchronises the host
    inside a chunk of iterations: once the device stop flag is raised every later kernel is a
    no-op (the collectives still run, identically on every rank), and the host reads the
    records and the executed count once per chunk, as ltb_pga_run does on one GPU."""
    lib, ctx = nat.lib(), nat.context()
    dt = m_rows.dtype
    if dt not in (torch.float32, torch.float64):
        m_rows = m_rows.double()
        dt = torch.float64
    code = nat.F32 if dt == torch.float32 else nat.F64
    r, I2 = int(m_rows.shape[0]), int(m_rows.shape[1])
    E = m_rows.numel()
    ntubes = r * I2
    P = engine.P
    dev = m_rows.device
    # every buffer handed to libltb by pointer is C-contiguous (a Fortran-ordered numpy mask,
    # e.g. sample_mask's, gives strided torch views and strided torch.where results)
    m_rows = m_rows.contiguous()
    mask_u8 = mask_rows.to(torch.uint8).contiguous()
    bits = torch.zeros(max((E + 31) // 32, 1), dtype=torch.int32, device=dev)
    nat.check(lib.ltb_pack_mask(ctx, E, mask_u8.data_ptr(), bits.data_ptr()))
    pobs = torch.where(mask_u8.bool(), m_rows, torch.zeros_like(m_rows)).contiguous()
    gt = gt_rows.to(dt).contiguous() if gt_rows is not None else None

    def allsum(vals):
        t = torch.as_tensor(vals, dtype=torch.float64, device=dev)
        dist.all_reduce(t, group=group)
        return t

    if mu0 is None and cfg.mu0 is None:
        mu0 = cfg.nu * math.sqrt(float(allsum([float((m_rows.double() ** 2).sum())])[0]))
    elif mu0 is None:
        mu0 = float(cfg.mu0)
    mus, ts, betas = pga_schedule(cfg, mu0)
    pobs_sumsq = float(allsum([float((pobs.double() ** 2).sum())])[0])
    gt_sumsq = None
    if gt is not None and cfg.rse_denominator == "original":
        gt_sumsq = float(allsum([float((gt.double() ** 2).sum())])[0])
    # the transform-domain dtype of the COMPUTE precision (as ltb_pga_run: complex of the real compute
    # dtype for complex specs), not apply_l's return dtype: the reference promotes an explicit-matrix
    # transform of float32 data to complex128, the fused PGA steps write complex64
    real_np = np.dtype(np.float32 if code == nat.F32 else np.float64)
    hat_np = np.dtype(nat.complex_of(real_np)) if engine.spec.is_complex else real_np
    hat_t = _TORCH_DT[hat_np]
    world, rank = _world(group)
    q0, q1 = blocks(P, world)[rank]
    nq, n = q1 - q0, min(I1, I2)
    xs = [torch.zeros_like(m_rows), torch.zeros_like(m_rows), torch.empty_like(m_rows)]
    hat_rows = torch.empty((P, r, I2), dtype=hat_t, device=dev)
    sl_out = torch.empty((nq, I1, I2), dtype=hat_t, device=dev)
    # carried right bases of this rank's slices: real domains, and complex64 slices too large for
    # the shared-memory Jacobi tier (I1 >= I2: ltb_svt_carry_c64_impl; smaller ones ignore it)
    carry_c = hat_t == torch.complex64 and I1 >= I2 and I1 * I2 * 8 > 200 * 1024
    vcarry = torch.empty((nq, n, n), dtype=hat_t if carry_c else dt, device=dev) \
        if nq and (not hat_t.is_complex or carry_c) else None
    state = torch.zeros(2, dtype=torch.int32, device=dev)
    sums = torch.zeros(5, dtype=torch.float64, device=dev)
    recs = torch.zeros((chunk, 5), dtype=torch.float64, device=dev)
    gt_ptr = gt.data_ptr() if gt is not None else None
    h = engine.handle.ptr
    trace = CompletionTrace()
    warm, done, ip, ic = 0, 0, 0, 1  # xs[ip] = x_prev, xs[ic] = x_cur
    k = 1
    while k <= cfg.max_iters and trace.status != "converged":
        count = min(chunk, cfg.max_iters - k + 1)
        nexts = []
        for i in range(count):
            kk = k + i
            inx = 3 - ip - ic
            xp, xc, xn = xs[ip], xs[ic], xs[inx]
            beta = float(betas[kk - 1])
            nat.check(lib.ltb_pga_shard_forward(ctx, h, code, ntubes, beta, xc.data_ptr(), xp.data_ptr(),
                                                pobs.data_ptr(), bits.data_ptr(), hat_rows.data_ptr(),
                                                state.data_ptr()))
            sl = fibres_to_slices(hat_rows, I1, group)
            nat.check(lib.ltb_pga_shard_svt(ctx, nat.dtype_code(hat_np), nq, I1, I2, sl.data_ptr(),
                                            float(mus[kk - 1]), sl_out.data_ptr(),
                                            vcarry.data_ptr() if vcarry is not None else None, warm,
                                            state.data_ptr()))
            warm = 1
            back = slices_to_fibres(sl_out, P, group)
            nat.check(lib.ltb_pga_shard_inverse(ctx, h, code, ntubes, beta, back.data_ptr(), xc.data_ptr(),
                                                xp.data_ptr(), gt_ptr, xn.data_ptr(), sums.data_ptr(),
                                                state.data_ptr()))
            dist.all_reduce(sums[:4], group=group)
            dist.all_reduce(sums[4:], op=dist.ReduceOp.MAX, group=group)
            nat.check(lib.ltb_pga_shard_decide(ctx, sums.data_ptr(), pobs_sumsq, float(cfg.tol),
                                               recs[i].data_ptr(), state.data_ptr()))
            nexts.append(inx)
            ip, ic = ic, inx
        st = state.tolist()
        rec = recs[:count].tolist()
        executed = st[1] - done
        for i in range(executed):
            kk = k + i
            r0, r1, r2, peak, _ = rec[i]
            rel = rel_change(r0, r1, pobs_sumsq == 0.0)
            item = IterationRecord(k=kk, mu=mus[kk - 1], t=ts[kk - 1], rel_change=rel)
            if gt is not None:
                den = math.sqrt(r1) ** 2 if cfg.rse_denominator == "obtained" else gt_sumsq
                err = math.sqrt(r2) ** 2
                item.rse = math.nan if den == 0.0 else err / den
                item.psnr = math.inf if err == 0.0 else (-math.inf if peak == 0.0 else
                                                         10.0 * math.log10(peak ** 2 / err))
            trace.records.append(item)
        done = st[1]
        if st[0]:
            trace.status = "converged"
            ic = nexts[executed - 1]  # the iterate of the last executed iteration
        k += count
    x_cur = xs[ic]
    out = torch.where(mask_u8.bool(), m_rows, x_cur).contiguous() if cfg.reimpose_observed else x_cur
    return out, trace


# ----------------------------------------------------------------- SPMD drop-in entry points
def _group(group):
    return None if isinstance(group, str) and group == "world" else group


def _gather_rows(x_rows: torch.Tensor, I1: int, group) -> np.ndarray:
    """All-gather the row blocks of a row-sharded tensor into the full (I1, ...) numpy array."""
    world, _ = _world(group)
    rb = blocks(I1, world)
    rmax = max(b - a for a, b in rb)
    buf = torch.zeros((rmax,) + tuple(x_rows.shape[1:]), dtype=x_rows.dtype, device=x_rows.device)
    buf[: x_rows.shape[0]] = x_rows
    allbuf = torch.empty((world * rmax,) + tuple(x_rows.shape[1:]), dtype=x_rows.dtype, device=x_rows.device)
    dist.all_gather_into_tensor(allbuf, buf, group=group)
    return torch.cat([allbuf[g * rmax: g * rmax + (b - a)] for g, (a, b) in enumerate(rb)]).cpu().numpy()


def _engine(spec, trailing):
    cache = spec.__dict__.setdefault("_spmd_engines", {})
    key = (tuple(int(d) for d in trailing), nat.current_device())
    if key not in cache:
        cache[key] = DeviceEngine(spec, trailing)
    return cache[key]


def spmd_pga_complete(m, mask, cfg: CompletionConfig, ground_truth=None, *, precision="fp64", group="world"):
    """pga_complete (completion.py:141-202) across the ranks of `group`, called by every rank
    with the same arguments (SPMD, one process per GPU under torchrun).  Rank g takes the
    i1-row block R_g; the iteration is dist_pga_complete's device path; every rank returns the
    full float64 iterate and the (identical) trace, as the single-process call does."""
    grp = _group(group)
    world, rank = _world(grp)
    from .core import fro_norm

    m64 = np.asarray(m, dtype=float)
    mask = np.asarray(mask, dtype=bool)
    I1 = m64.shape[0]
    r0, r1 = blocks(I1, world)[rank]
    dev = torch.device("cuda", nat.current_device())
    dt = torch.float32 if precision == "fp32" else torch.float64
    eng = _engine(cfg.spec, m64.shape[2:])
    m_rows = torch.from_numpy(np.ascontiguousarray(m64[r0:r1])).to(dev, dt)
    k_rows = torch.from_numpy(np.ascontiguousarray(mask[r0:r1])).to(dev)
    gt_rows = None
    if ground_truth is not None:
        gt_rows = torch.from_numpy(np.ascontiguousarray(np.asarray(ground_truth, dtype=float)[r0:r1])).to(dev, dt)
    mu0 = cfg.nu * fro_norm(m64) if cfg.mu0 is None else float(cfg.mu0)  # as the single-GPU call computes it
    x_rows, trace = dist_pga_complete(m_rows, k_rows, cfg, I1, eng, group=grp, ground_truth_rows=gt_rows, mu0=mu0)
    return _gather_rows(x_rows.double(), I1, grp), trace


def spmd_svt(a, tau: float, spec, *, group="world"):
    """svt (linalg.py:168-181) across the ranks of `group` (SPMD): row-sharded transforms, the
    slice-sharded SVT between two all-to-alls; every rank returns the full result."""
    grp = _group(group)
    world, rank = _world(grp)
    a = np.asarray(a)
    I1 = a.shape[0]
    r0, r1 = blocks(I1, world)[rank]
    dev = torch.device("cuda", nat.current_device())
    rows = torch.from_numpy(np.ascontiguousarray(a[r0:r1])).to(dev)
    out = dist_svt(rows, tau, I1, _engine(spec, a.shape[2:]), grp)
    return _gather_rows(out, I1, grp)


def spmd_l_product(a, b, spec, *, group="world"):
    """l_product (linalg.py:34-43) across the ranks of `group` (SPMD): rank g computes the rows
    R_g of C from its rows of A and all of B (rows of a *_L b depend only on the same rows of
    a), then the row blocks are all-gathered; every rank returns the full product."""
    from .linalg import l_product

    grp = _group(group)
    world, rank = _world(grp)
    a = np.asarray(a)
    I1 = a.shape[0]
    r0, r1 = blocks(I1, world)[rank]
    c_rows = l_product(np.ascontiguousarray(a[r0:r1]), b, spec)
    dev = torch.device("cuda", nat.current_device())
    return _gather_rows(torch.from_numpy(np.ascontiguousarray(c_rows)).to(dev), I1, grp)
