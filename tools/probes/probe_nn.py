import sys, os, torch
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
L = _lib.lib
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
m, n, k = 128, 256, 16
a = torch.zeros(m, k, device=dev)
for i in range(16): a[i, i] = 1.0
p = torch.arange(k, device=dev).float()[:, None]; j = torch.arange(n, device=dev).float()[None, :]
bt = (p * 1000 + j).contiguous()
c = torch.full((m, n), -1.0, device=dev)
_lib.check(L.mtnn_gemm_nn(a.data_ptr(), bt.data_ptr(), c.data_ptr(), m, n, k, 1, s)); torch.cuda.synchronize()
cc = c.cpu()
print("cfg", os.environ.get("MTNN_DEBUG_NN"))
for i in range(0, 16, 3):
    print(i, [int(x) for x in cc[i, :40:3].tolist()])
print("row 20", [int(x) for x in cc[20, :8].tolist()])
