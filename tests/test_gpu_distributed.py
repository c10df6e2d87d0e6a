"""The multi-GPU driver's device engine (distributed.DeviceEngine on libltb) through NCCL with
world_size 1 on cuda:0: the sharded l_product / SVT / PGA must reproduce the single-device
API.  (More ranks than GPUs are never emulated on one GPU; the exchanges themselves are
covered for world 2/3 by tests/test_distributed.py with gloo.)"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2202_02870_b200 as L
from paper_2202_02870_b200.distributed import (DeviceEngine, DistLProductPlan, dist_l_product, dist_pga_complete,
                                               dist_svt)
from ltb_testutil import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_dist_l_product_device(nccl_world1):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((64, 16, 3, 8)).astype(np.float32)
    b = rng.standard_normal((16, 48, 3, 8)).astype(np.float32)
    spec = L.make_spec("dct", (64, 48, 3, 8))
    eng = DeviceEngine(spec, (3, 8))
    c = dist_l_product(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), eng)
    torch.cuda.synchronize()
    assert rel_err(c.cpu().numpy(), L.l_product(a, b, spec)) < 1e-5


@pytest.mark.parametrize("transform,dtype,tol", [("dct", np.float32, 1e-5), ("fft", np.float64, 1e-10)])
def test_dist_plan_exchange_device(nccl_world1, transform, dtype, tol):
    """The plan with its NCCL all-gather + permute kept at world 1, preallocated output."""
    rng = np.random.default_rng(8)
    a = rng.standard_normal((40, 24, 4, 6)).astype(dtype)
    b = rng.standard_normal((24, 36, 4, 6)).astype(dtype)
    spec = L.make_spec(transform, (40, 36, 4, 6))
    eng = DeviceEngine(spec, (4, 6))
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    plan = DistLProductPlan(ta.shape, tb.shape, eng, ta.dtype, ta.device, exchange=True)
    out = torch.empty(plan.c_shape, dtype=ta.dtype, device="cuda")
    for _ in range(2):  # buffers are reused across runs
        plan.run(ta, tb, out=out)
    torch.cuda.synchronize()
    assert rel_err(out.cpu().numpy(), L.l_product(a, b, spec)) < tol


def test_dist_svt_device(nccl_world1):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((20, 12, 6))
    spec = L.make_spec("fft", x.shape)
    out = dist_svt(torch.from_numpy(x).cuda(), 0.9, 20, DeviceEngine(spec, (6,)))
    torch.cuda.synchronize()
    assert rel_err(out.cpu().numpy(), L.svt(x, 0.9, spec)) < 1e-10


def test_dist_pga_device(nccl_world1, golden):
    m = golden["c_dct/m"]
    mask = golden["c_dct/mask"]
    spec = L.make_spec("dct", m.shape)
    cfg = L.CompletionConfig(spec=spec, max_iters=30)
    x, trace = dist_pga_complete(torch.from_numpy(m).cuda(), torch.from_numpy(mask).cuda(), cfg, m.shape[0],
                                 DeviceEngine(spec, m.shape[2:]))
    ref, rtrace = L.pga_complete(m, mask, cfg)
    assert trace.iterations == rtrace.iterations
    assert rel_err(x.cpu().numpy(), ref) < 1e-10


def test_dist_pga_fp32_carried_device(nccl_world1):
    """fp32 slices of width >= 32 take the warm-started SVT (ltb_slice_svt_carry) and the
    device-side norms; the iterate must match the single-device fp32 solver within the fp32
    tolerance after enough iterations for every slice to be solved."""
    rng = np.random.default_rng(12)
    a = rng.standard_normal((48, 4, 3, 5))
    b = rng.standard_normal((4, 40, 3, 5))
    spec = L.make_spec("dct", (48, 40, 3, 5))
    x0 = L.l_product(a, b, spec)
    m = x0.astype(np.float32)
    mask = rng.random(m.shape) < 0.5
    cfg = L.CompletionConfig(spec=spec, max_iters=60, tol=1e-300)
    mu0 = cfg.nu * float(np.linalg.norm(m.astype(np.float64)))
    x, trace = dist_pga_complete(torch.from_numpy(m).cuda(), torch.from_numpy(mask).cuda(), cfg, m.shape[0],
                                 DeviceEngine(spec, m.shape[2:]), mu0=mu0)
    ref, rtrace = L.pga_complete(m.astype(np.float64), mask, cfg)
    assert trace.iterations == rtrace.iterations == 60
    assert rel_err(x.cpu().numpy(), ref) < 1e-4


def test_dist_pga_complex_carried_device(nccl_world1):
    """Complex64 slices beyond the shared-memory Jacobi tier (config 4's recipe at 256 x 256 x 3 x 8):
    the sharded PGA step carries V^T per rank (ltb_pga_shard_svt -> the carried blocked Jacobi with
    truncated sweeps, no conjugate mirroring across ranks); the iterate must match the single-device
    solver, which mirrors conjugate slice pairs, within the fp32 tolerance."""
    rng = np.random.default_rng(0)
    shape = (256, 256, 3, 8)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    spec = L.make_spec("explicit", shape, matrices={3: q, 4: L.build_fourier_matrix(8)})
    a = rng.standard_normal((256, 8, 3, 8), dtype=np.float32)
    b = rng.standard_normal((8, 256, 3, 8), dtype=np.float32)
    m = L.l_product(a, b, spec).astype(np.float32)
    mask = rng.random(m.shape) < 0.3
    cfg = L.CompletionConfig(spec=spec, max_iters=40, tol=1e-300)
    mu0 = cfg.nu * float(np.linalg.norm(m.astype(np.float64)))
    x, trace = dist_pga_complete(torch.from_numpy(m).cuda(), torch.from_numpy(mask).cuda(), cfg, m.shape[0],
                                 DeviceEngine(spec, m.shape[2:]), mu0=mu0)
    ref, rtrace = L.pga_complete(m, mask, cfg)
    assert trace.iterations == rtrace.iterations == 40
    assert np.count_nonzero(ref) > 0
    assert rel_err(x.cpu().numpy(), ref) < 1e-4


def test_dist_pga_device_converges_midchunk(nccl_world1, golden):
    """The device stop flag: a default-tol run that converges inside a chunk returns the
    iterate of the converging iteration and the same trace as the single-device solver."""
    name = "c_pinned_dct"
    m = golden[f"{name}/m"]
    spec = L.make_spec("dct", m.shape)
    mask = L.sample_mask(m.shape, 0.5, 7)
    cfg = L.CompletionConfig(spec=spec, max_iters=300)
    x, trace = dist_pga_complete(torch.from_numpy(m).cuda(), torch.from_numpy(mask).cuda(), cfg, m.shape[0],
                                 DeviceEngine(spec, m.shape[2:]))
    ref, rtrace = L.pga_complete(m, mask, cfg)
    assert trace.status == rtrace.status == "converged"
    assert trace.iterations == rtrace.iterations
    np.testing.assert_allclose([r.rel_change for r in trace.records], [r.rel_change for r in rtrace.records],
                               rtol=1e-8)
    assert rel_err(x.cpu().numpy(), ref) < 1e-10


def test_spmd_drop_in_entry_points(nccl_world1, golden):
    """The reference entry points with group="world": every rank makes the same call and gets
    the full result (here world 1: the sharded path end to end through NCCL)."""
    m = golden["c_gt/m"]
    mask = golden["c_gt/mask"]
    spec = L.make_spec("fft", m.shape)
    cfg = L.CompletionConfig(spec=spec, max_iters=15, tol=1e-12, reimpose_observed=True)
    x, trace = L.pga_complete(m, mask, cfg, ground_truth=m, group="world")
    ref, rtrace = L.pga_complete(m, mask, cfg, ground_truth=m)
    assert x.dtype == np.float64 and x.shape == m.shape
    assert trace.iterations == rtrace.iterations
    np.testing.assert_allclose([r.rse for r in trace.records], [r.rse for r in rtrace.records], rtol=1e-8)
    assert rel_err(x, ref) < 1e-10
    rng = np.random.default_rng(21)
    a = rng.standard_normal((30, 7, 3, 4))
    b = rng.standard_normal((7, 20, 3, 4))
    pspec = L.make_spec("dct", (30, 20, 3, 4))
    assert rel_err(L.l_product(a, b, pspec, group="world"), L.l_product(a, b, pspec)) < 1e-12
    xs = rng.standard_normal((18, 14, 5))
    sspec = L.make_spec("fft", xs.shape)
    assert rel_err(L.svt(xs, 0.7, sspec, group="world"), L.svt(xs, 0.7, sspec)) < 1e-10
