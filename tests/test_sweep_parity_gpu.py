"""The whole headline configuration (configs[1]: m, n, k in {2^7..2^14}, 512
shapes) through the MTNN dispatcher with the shipped B200 model, on the
reference harness's operands make_operands(shape, 0) (pkg/src/mtnn/bench.py:
104-114, generated on the device bit-identically), checked against float64 on a
sampled 16 x 16 block of every output — plus the forced-TNN path, and the NT
branch bit-identical to a direct gemm_nt (the dispatcher adds no arithmetic)."""

import numpy as np
import pytest
import torch

from paper_1702_03192_b200 import device, gbdt, operands
from paper_1702_03192_b200.platform import probe_platform
from paper_1702_03192_b200.selector import Choice, Dispatcher

pytestmark = pytest.mark.gpu

FP32_GATE = 1e-5
MODEL = __import__("pathlib").Path(__file__).resolve().parent.parent / \
    "paper_1702_03192_b200" / "models" / "b200_sweep.json"


def test_all_512_sweep_shapes_through_the_dispatcher():
    sizes = [2 ** e for e in range(7, 15)]
    stream = operands.operand_stream(2 * 16384 * 16384, seed=0)
    disp = Dispatcher(gbdt.load_model(str(MODEL)), probe_platform())
    rng = np.random.default_rng(0)
    worst, tnn_cases = 0.0, 0
    for m in sizes:
        for n in sizes:
            for k in sizes:
                a, b = operands.views(stream, m, n, k)
                c = disp.gemm(a, b)
                chose_tnn = disp.last_choice == Choice.USE_TNN
                tnn_cases += chose_tnn
                rows = np.sort(rng.choice(m, 16, replace=False))
                cols = np.sort(rng.choice(n, 16, replace=False))
                ar = a[torch.from_numpy(rows).cuda()].double().cpu().numpy()
                bc = b[torch.from_numpy(cols).cuda()].double().cpu().numpy()
                want = ar @ bc.T
                ct = device.gemm_tnn(a, b)
                for name, got in (("mtnn", c), ("tnn", ct)):
                    g = got[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()]
                    g = g.double().cpu().numpy()
                    err = np.linalg.norm(g - want) / np.linalg.norm(want)
                    worst = max(worst, err)
                    assert err < FP32_GATE, ((m, n, k), name, err)
                if not chose_tnn:  # the NT branch is exactly gemm_nt
                    assert torch.equal(c, device.gemm_nt(a, b)), (m, n, k)
    print(f"512 shapes: worst sampled rel. Frobenius {worst:.2e}; TNN chosen {tnn_cases}x")
