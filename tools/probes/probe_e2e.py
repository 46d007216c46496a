"""Time one e2e sweep pass through mtnn_dispatch_gemm_host with pinned buffers."""
import ctypes, os, sys, time
import torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib, gbdt
from paper_1702_03192_b200.platform import probe_platform
from paper_1702_03192_b200.selector import Dispatcher
L = _lib.lib
torch.cuda.set_device(0)
shapes = [(m, n, k) for m in [2**e for e in range(7, 15)] for n in [2**e for e in range(7, 15)] for k in [2**e for e in range(7, 15)]]
d = Dispatcher(gbdt.GbdtModel(trees=(), params=gbdt.GbdtParams(), n_features=8), probe_platform())
mx = 16384 * 16384
ha = torch.empty(mx).pin_memory(); hb = torch.empty(mx).pin_memory(); hc = torch.empty(mx).pin_memory()
ha.uniform_(-1, 1); hb.uniform_(-1, 1)
ch = ctypes.c_int()
def step(sub):
    for (m, n, k) in sub:
        _lib.check(L.mtnn_dispatch_gemm_host(d._native.handle, d._prefix_p, ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, -1, 0, ctypes.byref(ch)))
step(shapes[:64]); step(shapes[-8:])
t0 = time.perf_counter(); step(shapes); dt = time.perf_counter() - t0
fl = sum(2.0 * m * n * k for m, n, k in shapes)
print(f"{os.environ.get('MTNN_PIPE_MIN_MB','48')} MB min, {os.environ.get('MTNN_PIPE_CHUNK_MB','16')} MB chunk: e2e {fl/dt/1e12:.1f} TF ({dt:.3f} s)", flush=True)
big = [(16384, 16384, 16384)]
t0 = time.perf_counter(); step(big); dt = time.perf_counter() - t0
print(f"   16384^3 alone: {dt*1e3:.1f} ms (3 GiB over PCIe: {3*2**30/dt/1e9:.1f} GB/s)")
