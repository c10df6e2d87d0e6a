"""Host-link rate of 2-D strided copies (rows of W bytes at a host pitch of 2 W) against 1-D
copies of the same bytes, pinned host memory, each direction alone and both at once."""
import time
import torch
from cuda.bindings import runtime as rt

MB = 1 << 20
dev = torch.empty(64 * MB, dtype=torch.uint8, device="cuda")
host = torch.empty(128 * MB, dtype=torch.uint8, pin_memory=True)
dev2 = torch.empty(64 * MB, dtype=torch.uint8, device="cuda")
host2 = torch.empty(128 * MB, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


def copy(kind, width, rows, stream, two_d, dst_off=0):
    if kind == H2D:
        d, h = dev2.data_ptr(), host2.data_ptr()
        if two_d:
            return rt.cudaMemcpy2DAsync(d, width, h, 2 * width, width, rows, kind, stream.cuda_stream)
        return rt.cudaMemcpyAsync(d, h, width * rows, kind, stream.cuda_stream)
    d, h = dev.data_ptr(), host.data_ptr()
    if two_d:
        return rt.cudaMemcpy2DAsync(h, 2 * width, d, width, width, rows, kind, stream.cuda_stream)
    return rt.cudaMemcpyAsync(h, d, width * rows, kind, stream.cuda_stream)


for width in (12 * 1024, 24 * 1024, 48 * 1024, 96 * 1024):
    rows = (24 * MB) // width
    for two_d in (False, True):
        res = []
        for mode in ("h2d", "d2h", "both"):
            for _ in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if mode in ("h2d", "both"):
                    copy(H2D, width, rows, s1, two_d)
                if mode in ("d2h", "both"):
                    copy(D2H, width, rows, s2, two_d)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
            res.append(f"{mode} {width * rows / dt / 1e9:5.1f} GB/s")
        print(f"width {width // 1024:3d} KB {'2D' if two_d else '1D'}: " + ", ".join(res), flush=True)
