for rep in 1 2; do for v in default noitems; do
  lib=$PWD/paper_1702_03192_b200/lib/libmtnn_b200.so; [ $v = noitems ] && lib=$PWD/build/variants/noitems/libmtnn_b200.so
  MTNN_B200_LIB=$lib timeout 600 python bench.py --workload single --steps 20 --warmup 5 --no-cpu --no-e2e --no-verify 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v single',round(d['ms_per_step']*1e3,1),'us')"
done; done
python - <<'P'
import sys, torch, ctypes
sys.path.insert(0, ".")
from paper_1702_03192_b200 import _lib
import numpy as np
# how many entries does a 1024^3 call list on the bench operands?
from paper_1702_03192_b200 import operands as ops
A = ops.operand_stream(2 * 1024 * 1024, seed=0, device=torch.device("cuda"))
a = A[:1024*1024].view(1024,1024).cpu().numpy(); b = A[1024*1024:].view(1024,1024).cpu().numpy()
for x, nm in ((a, "A"), (b, "B")):
    mx = np.abs(x).max(axis=1, keepdims=True)
    print(nm, "elements below 2^-20 of their row max:", int((np.abs(x) < mx * 2.0**-20).sum()), "min |x|", float(np.abs(x).min()))
P
