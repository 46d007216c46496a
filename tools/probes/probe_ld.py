import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_1702_03192_b200 import gemm_nt
m = n = k = int(sys.argv[1])
torch.manual_seed(0)
a = torch.rand(m, k, device="cuda") * 2 - 1; b = torch.rand(n, k, device="cuda") * 2 - 1
c = gemm_nt(a, b); c = gemm_nt(a, b); torch.cuda.synchronize()
rows = np.arange(0, m, 251); cols = np.arange(0, n, 241)
want = oracle.oracle_nt_rows(a.cpu().numpy(), b.cpu().numpy(), rows, cols)
print("err", oracle.rel_frobenius(c.cpu().numpy()[np.ix_(rows, cols)], want))
