import ctypes, time, torch
dev = torch.device("cuda:0")
cudart = ctypes.CDLL("libcudart.so") if False else None
N = 256 * 2**20
h = torch.empty(N, dtype=torch.float32).pin_memory()
d = torch.empty(N, device=dev)
s = torch.cuda.Stream()
import cuda.bindings.runtime as rt
def copy2d(rows, width_f, pitch_f, reps=5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in range(reps):
        err, = rt.cudaMemcpy2DAsync(h.data_ptr(), pitch_f * 4, d.data_ptr(), width_f * 4, width_f * 4, rows,
                                    rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s.cuda_stream)
    s.synchronize()
    return rows * width_f * 4 * reps / (time.perf_counter() - t0) / 1e9
for (rows, w, p) in [(2048, 2048, 16384), (2048, 2048, 2048), (4096, 2048, 16384), (1024, 4096, 16384), (2048, 8192, 16384), (16384, 512, 16384)]:
    print(f"D2H 2D rows={rows} width={w*4}B pitch={p*4}B: {copy2d(rows, w, p):.1f} GB/s")
