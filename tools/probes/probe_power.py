"""Board power and SM clock while one kernel class runs back to back for ~3 s:
the operand split (HBM-bound) vs the tc3xf16s GEMM (tensor-bound)."""
import subprocess, sys, threading, time, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
A = torch.rand(16384 * 16384, device=dev); B = torch.rand(16384 * 16384, device=dev); C = torch.empty(16384 * 16384, device=dev)
def sample(stop, out):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits", "-lms", "100"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line: out.append([float(x) for x in line.split(",")])
    p.terminate()
def run(name, fn, secs=3.0):
    fn(); torch.cuda.synchronize()
    stop = threading.Event(); out = []
    th = threading.Thread(target=sample, args=(stop, out)); th.start()
    time.sleep(0.3)
    t0 = time.time(); n = 0
    while time.time() - t0 < secs:
        for _ in range(4): fn()
        torch.cuda.synchronize(); n += 4
    stop.set(); th.join()
    load = out[3:-1] or out
    pw = sorted(x[0] for x in load); ck = sorted(x[1] for x in load)
    print(f"{name}: {n} calls, power median {pw[len(pw)//2]:.0f} W max {pw[-1]:.0f} W, sm clock median {ck[len(ck)//2]:.0f} MHz", flush=True)
wa = torch.empty(16384 * 16384 * 2 + 16384 * 2, dtype=torch.float16, device=dev)
inv = torch.empty(16384, device=dev)
h = wa[: 16384 * 16384]; l = wa[16384 * 16384: 2 * 16384 * 16384]
run("split 16384x16384 (1 GiB -> h/l)", lambda: _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), 16384, 128, 16384, 3, s)) if False else None)
import ctypes
lib = ctypes.CDLL(str(_lib.LIB_PATH))
# operand split alone through a GEMM with tiny n/m would include GEMM work; use the transpose as the HBM-bound stand-in too
run("transpose 16384^2 (HBM-bound copy)", lambda: _lib.check(L.mtnn_transpose(A.data_ptr(), C.data_ptr(), 16384, 16384, s)))
run("gemm tc3xf16s 8192^3", lambda: _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), 8192, 8192, 8192, 3, s)))
run("gemm tc3xf16s 16384x16384x16384", lambda: _lib.check(L.mtnn_gemm_nt(A.data_ptr(), B.data_ptr(), C.data_ptr(), 16384, 16384, 16384, 3, s)), secs=4.0)
