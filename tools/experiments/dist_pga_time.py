"""Config-3 PGA through distributed.dist_pga_complete (run under torchrun, one rank per GPU):
iterations/s (device-synchronised wall time, max over ranks)."""
import os
import sys
import time
from pathlib import Path
import numpy as np
import torch
import torch.distributed as dist
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2202_02870_b200 as L  # noqa: E402
from paper_2202_02870_b200 import _native as nat  # noqa: E402
from paper_2202_02870_b200.distributed import DeviceEngine, blocks, dist_pga_complete  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ws, rank = dist.get_world_size(), dist.get_rank()
nat.set_device(local)
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
m, mask = bench._cfg3_data_host()
spec = L.make_spec("dct", bench.CFG3["shape"])
r0, r1 = blocks(m.shape[0], ws)[rank]
mu0 = 0.9 * float(np.linalg.norm(m.astype(np.float64)))
eng = DeviceEngine(spec, m.shape[2:])
mt = torch.from_numpy(np.ascontiguousarray(m[r0:r1])).cuda()
kt = torch.from_numpy(np.ascontiguousarray(mask[r0:r1])).cuda()
for n in (3, iters):
    cfg = L.CompletionConfig(spec=spec, tol=1e-300, max_iters=n)
    torch.cuda.synchronize(); dist.barrier()
    t0 = time.perf_counter()
    x, trace = dist_pga_complete(mt, kt, cfg, m.shape[0], eng, mu0=mu0)
    torch.cuda.synchronize()
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
if rank == 0:
    print(f"world {ws}: {iters} iterations in {float(t[0]):.3f} s -> {iters / float(t[0]):.1f} it/s", flush=True)
dist.destroy_process_group()
