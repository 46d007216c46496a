"""GPU parity of the kernel API against the oracle and the reference's golden
outputs. Mirrors /root/reference/pkg/tests/test_kernels.py (KATs, bit-exact
identities, oracle <= 1e-4 on random shapes, transpose involution, cross-kernel
equivalence, inputs never mutated) and adds the B200 gates: rel-Frobenius
<= 1e-5 vs float64 for FP32 GEMMs at large shapes, bit-exact transposes of
raw bit patterns (NaN payloads, -0.0) on every path."""

import numpy as np
import pytest

import oracle
from oracle import random_matrix, rel_frobenius
from paper_1702_03192_b200 import kernels
from paper_1702_03192_b200.kernels import as_matrix, gemm_nn, gemm_nt, gemm_tnn, transpose_oop

pytestmark = pytest.mark.gpu

TOL = 1e-4          # reference tolerance (test_kernels.py:17)
FP32_GATE = 1e-5    # north_star: rel Frobenius vs float64-accumulated result
VARIANTS = ("auto", "tc3xf16s", "tc3xtf32", "ffma")


def eye(n):
    return np.eye(n, dtype=np.float32)


def tc_ok(m, n, k, v="tc3xtf32"):
    return k % 4 == 0 and n % 4 == 0 and (v != "tc3xf16s" or k % 8 == 0)


class TestKats:
    def test_one_by_one(self):
        assert gemm_nn(as_matrix([[2.0]]), as_matrix([[3.0]]))[0, 0] == 6.0

    def test_dot_product(self):
        assert gemm_nt(as_matrix([[1.0, 2.0]]), as_matrix([[3.0, 4.0]]))[0, 0] == 11.0

    def test_transpose_definition(self):
        b = as_matrix([[1.0, 2.0, 3.0], [4.0, 5.0, 6.0]])
        assert np.array_equal(transpose_oop(b), np.array([[1, 4], [2, 5], [3, 6]], np.float32))

    def test_scalar_tnn(self):
        assert gemm_tnn(as_matrix([[2.0]]), as_matrix([[-3.0]]))[0, 0] == -6.0

    def test_golden_kats(self, golden_kernels):
        g = golden_kernels
        assert np.array_equal(transpose_oop(g["kat_t_in"]), g["kat_t_out"])
        assert np.array_equal(gemm_nn(g["ident_a"], eye(130), block=64), g["ident_nn"])
        assert np.array_equal(gemm_nt(g["ident_a"][:3, :3].copy(), eye(3)), g["ident_nt"])


class TestIdentities:
    def test_identity_times_b(self, rng):
        b = random_matrix(rng, 3, 4)
        assert np.array_equal(gemm_nn(eye(3), b), b)

    def test_b_identity_bitexact(self, rng):
        for m, k in ((3, 3), (70, 70), (130, 130)):
            a = random_matrix(rng, m, k)
            assert np.array_equal(gemm_nn(a, eye(k), block=64), a)
            assert np.array_equal(gemm_nt(a, eye(k)), a)
            assert np.array_equal(gemm_tnn(a, eye(k)), a)

    def test_ffma_identity_bitexact_any_size(self, rng):
        a = random_matrix(rng, 300, 260)
        assert np.array_equal(gemm_nt(a, eye(260), variant="ffma"), a)

    def test_tc_identity_close(self, rng):
        a = random_matrix(rng, 256, 256)
        assert rel_frobenius(gemm_nt(a, eye(256), variant="tc3xtf32"), a) < 1e-6
        assert rel_frobenius(gemm_nt(a, eye(256), variant="tc3xf16s"), a) < 1e-6


class TestScaledF16Robustness:
    """tc3xf16s: per-row power-of-two scaling keeps FP32 accuracy across magnitudes
    FP16 cannot represent, and non-finite inputs propagate like FP32."""

    def test_wide_dynamic_range(self, rng):
        m, n, k = 384, 272, 520
        # rows spanning e^-40..e^40 (A) and e^-20..e^20 (B): far outside FP16's range,
        # products still inside FP32's
        a = (rng.standard_normal((m, k)) * np.exp(rng.uniform(-40, 40, (m, 1)))).astype(np.float32)
        b = (rng.standard_normal((n, k)) * np.exp(rng.uniform(-20, 20, (n, 1)))).astype(np.float32)
        want = oracle.oracle_nt_blas(a, b)
        for fn, bb in ((gemm_nt, b), (gemm_nn, np.ascontiguousarray(b.T))):
            got = fn(a, bb, variant="tc3xf16s")
            # relative error of every (row-block, column-block) — magnitudes differ by e^120
            rel = np.abs(got - want) / (np.linalg.norm(a.astype(np.float64), axis=1)[:, None]
                                        * np.linalg.norm(b.astype(np.float64), axis=1)[None, :])
            assert rel.max() < 1e-6
            err = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
            assert err.max() < FP32_GATE

    def test_zero_rows_and_nonfinite(self, rng):
        a = random_matrix(rng, 256, 256)
        b = random_matrix(rng, 256, 256)
        a[3] = 0.0
        a[5, 7] = np.inf
        a[9, 1] = np.nan
        got = gemm_nt(a, b, variant="tc3xf16s")
        want = oracle.oracle_nt_blas(a, b)
        assert np.all(got[3] == 0.0)
        assert np.all(~np.isfinite(got[5])) and np.all(np.isnan(got[9]))
        ok = np.ones(256, bool); ok[[5, 9]] = False
        assert rel_frobenius(got[ok], want[ok]) < FP32_GATE


class TestAgainstGolden:
    def test_all_golden_shapes_all_variants(self, golden_kernels):
        g = golden_kernels
        for i, (m, n, k) in enumerate(g["shapes"]):
            a, b, f64 = g[f"a{i}"], g[f"b{i}"], g[f"f64_{i}"]
            bt = np.ascontiguousarray(b.T)
            assert np.array_equal(transpose_oop(b), g[f"t{i}"])
            for v in VARIANTS:
                if v.startswith("tc") and not tc_ok(m, n, k, v):
                    continue
                for got in (gemm_nt(a, b, variant=v), gemm_tnn(a, b, variant=v)):
                    assert rel_frobenius(got, f64) < FP32_GATE
                    assert rel_frobenius(got, g[f"nt{i}"]) < FP32_GATE
                if not v.startswith("tc") or n % 16 == 0:
                    assert rel_frobenius(gemm_nn(a, bt, variant=v), g[f"nn{i}"]) < FP32_GATE

    def test_bit_patterns(self, golden_kernels):
        bits = golden_kernels["bits_in"]
        out = transpose_oop(bits.view(np.float32)).view(np.uint32)
        assert np.array_equal(out, golden_kernels["bits_out"])


class TestRandomAgainstOracle:
    def test_random_small_shapes(self, rng):
        for _ in range(50):
            m, n, k = (int(v) for v in rng.integers(1, 65, size=3))
            a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
            want = oracle.oracle_nt(a, b)
            assert rel_frobenius(gemm_nt(a, b), want) < TOL
            assert rel_frobenius(gemm_tnn(a, b), want) < TOL
            assert rel_frobenius(gemm_nn(a, np.ascontiguousarray(b.T)), want) < TOL

    def test_exhaustive_small(self, rng):
        sizes = (1, 2, 3, 5, 8, 17)
        for m in sizes:
            for n in sizes:
                for k in sizes:
                    a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
                    want = oracle.oracle_nt(a, b)
                    assert rel_frobenius(gemm_nt(a, b), want) < TOL
                    assert rel_frobenius(gemm_tnn(a, b), want) < TOL
                    assert rel_frobenius(gemm_nn(a, transpose_oop(b)), want) < TOL

    def test_acceptance_grid(self, rng):
        # reference acceptance criterion 1 (test_acceptance.py:68-88) at the FP32 gate
        for m in (1, 17, 64):
            for n in (1, 17, 64):
                for k in (1, 17, 64):
                    a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
                    want = oracle.oracle_nt(a, b)
                    assert rel_frobenius(gemm_nt(a, b), want) < FP32_GATE
                    assert rel_frobenius(gemm_tnn(a, b), want) < FP32_GATE

    @pytest.mark.parametrize("shape", [(128, 128, 128), (256, 512, 128), (200, 300, 100),
                                       (130, 260, 36), (1000, 1000, 1000), (4097, 1023, 260),
                                       (512, 10, 4096), (10, 4096, 1024), (1024, 4096, 784)])
    def test_mid_shapes_every_variant(self, rng, shape):
        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        want = oracle.oracle_nt_blas(a, b)
        bt = np.ascontiguousarray(b.T)
        for v in VARIANTS:
            if v.startswith("tc") and not tc_ok(m, n, k, v):
                continue
            assert rel_frobenius(gemm_nt(a, b, variant=v), want) < FP32_GATE, v
            if not v.startswith("tc") or n % 16 == 0:
                assert rel_frobenius(gemm_nn(a, bt, variant=v), want) < FP32_GATE, v
                assert rel_frobenius(gemm_tnn(a, b, variant=v), want) < FP32_GATE, v


class TestTranspose:
    def test_involution_bitexact(self, rng):
        for _ in range(20):
            r, c = (int(v) for v in rng.integers(1, 300, size=2))
            b = random_matrix(rng, r, c)
            assert np.array_equal(transpose_oop(transpose_oop(b)), b)

    @pytest.mark.parametrize("shape", [(1, 1), (2, 3), (37, 65), (128, 128), (1000, 1000),
                                       (3000, 5000), (16384, 128), (128, 16384), (4097, 1023),
                                       (8191, 8193), (64, 4), (4, 64)])
    def test_random_bits_bitexact(self, rng, shape):
        b = oracle.random_bits(rng, *shape)
        out = transpose_oop(b)
        assert out.shape == shape[::-1]
        assert np.array_equal(out.view(np.uint32), b.view(np.uint32).T)

    def test_fresh_buffer(self, rng):
        b = random_matrix(rng, 4, 4)
        out = transpose_oop(b)
        assert out.base is None or out.base is not b


class TestCrossKernel:
    def test_inputs_never_mutated(self, rng):
        a, b = random_matrix(rng, 40, 30), random_matrix(rng, 20, 30)
        a0, b0 = a.copy(), b.copy()
        gemm_nt(a, b); gemm_tnn(a, b); transpose_oop(b); gemm_nn(a, transpose_oop(b))
        assert np.array_equal(a, a0) and np.array_equal(b, b0)

    def test_result_dtype_and_layout(self, rng):
        c = gemm_nn(random_matrix(rng, 5, 7), random_matrix(rng, 7, 2))
        assert c.dtype == np.float32 and c.flags.c_contiguous

    def test_mem_budget(self, rng):
        a, b = random_matrix(rng, 8, 8), random_matrix(rng, 8, 8)
        with pytest.raises(MemoryError, match="budget"):
            gemm_tnn(a, b, mem_budget=16)
        gemm_tnn(a, b, mem_budget=10**9)

    def test_threads_argument_is_accepted(self, rng):
        a, b = random_matrix(rng, 80, 60), random_matrix(rng, 70, 60)
        assert rel_frobenius(gemm_nt(a, b, threads=2), gemm_nt(a, b)) < 1e-6


class TestDeviceTensors:
    def test_device_paths_match_host_paths(self, rng):
        import torch

        a, b = random_matrix(rng, 300, 200), random_matrix(rng, 256, 200)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        want = oracle.oracle_nt_blas(a, b)
        for v in VARIANTS:
            assert rel_frobenius(gemm_nt(ta, tb, variant=v).cpu().numpy(), want) < FP32_GATE
            assert rel_frobenius(gemm_tnn(ta, tb, variant=v).cpu().numpy(), want) < FP32_GATE
            tbt = transpose_oop(tb)
            assert torch.equal(tbt, tb.t().contiguous())
            assert rel_frobenius(gemm_nn(ta, tbt, variant=v).cpu().numpy(), want) < FP32_GATE

    def test_device_transpose_bits(self, rng):
        import torch

        b = oracle.random_bits(rng, 1000, 4000)
        tb = torch.from_numpy(b.view(np.int32)).cuda().view(torch.float32)
        out = transpose_oop(tb).view(torch.int32).cpu().numpy().view(np.uint32)
        assert np.array_equal(out, b.view(np.uint32).T)


class TestPipelinedHostPath:
    """Large numpy calls run the chunked H2D / compute / D2H pipeline inside the
    C-ABI (mtnn_*_host); results must match the device path and the oracle."""

    @pytest.mark.parametrize("shape", [(3000, 2048, 4096), (4096, 1000, 2048), (257, 8192, 4096),
                                       (2304, 16384, 1024)])  # (A-first prefix of the blocked pipeline)
    def test_pipelined_matches(self, rng, shape):
        import torch

        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        rows = np.sort(rng.choice(m, 64, replace=False))
        want = oracle.oracle_nt_rows(a, b, rows, np.arange(n))
        for fn in (gemm_nt, gemm_tnn):
            got = fn(a, b)
            assert rel_frobenius(got[rows], want) < FP32_GATE
        got = gemm_nn(a, np.ascontiguousarray(b.T))
        assert rel_frobenius(got[rows], want) < FP32_GATE
        dev = gemm_nt(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
        assert rel_frobenius(gemm_nt(a, b), dev) < 1e-6


    @pytest.mark.parametrize("shape", [(2304, 16384, 1024), (1024, 4096, 4096)])
    def test_blocked_pipeline_sm_stores_match_copies(self, rng, shape):
        """host_pipeline_zc: the blocked pipeline's C blocks written by SM stores
        into the pinned (device-mapped) host C — the same bits as the copy-engine
        2-D copies."""
        import torch

        from paper_1702_03192_b200 import _lib

        m, n, k = shape
        ha = torch.from_numpy(random_matrix(rng, m, k)).pin_memory()
        hb = torch.from_numpy(random_matrix(rng, n, k)).pin_memory()
        outs = []
        old = _lib.config_get("host_pipeline_zc")
        try:
            for v in (0, 1):
                _lib.config_set("host_pipeline_zc", v)
                hc = torch.full((m, n), float("nan")).pin_memory()
                _lib.check(_lib.lib.mtnn_gemm_nt_host(ha.data_ptr(), hb.data_ptr(), hc.data_ptr(), m, n, k, 0))
                outs.append(hc.numpy().copy())
        finally:
            _lib.config_set("host_pipeline_zc", old)
        assert np.array_equal(outs[0], outs[1])
        rows = np.sort(rng.choice(m, 32, replace=False))
        want = oracle.oracle_nt_rows(ha.numpy(), hb.numpy(), rows, np.arange(n))
        assert rel_frobenius(outs[1][rows], want) < FP32_GATE


def test_tf32_inkernel_split_opt_in(tmp_path):
    """MTNN_TF32_INKERNEL=1: the TF32 kernel computes the larger operand's lo half
    in shared memory; results stay within the FP32 gate (fresh process: the
    switch is read once)."""
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import numpy as np, oracle\n"
        "from paper_1702_03192_b200 import gemm_nt, gemm_nn\n"
        "rng = np.random.default_rng(3)\n"
        "for m, n, k in ((1024, 256, 2048), (256, 1024, 2048), (2048, 2048, 512)):\n"
        "    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)\n"
        "    b = rng.uniform(-1, 1, (n, k)).astype(np.float32)\n"
        "    want = oracle.oracle_nt_blas(a, b)\n"
        "    assert oracle.rel_frobenius(gemm_nt(a, b, variant='tc3xtf32'), want) < 1e-5\n"
        "    assert oracle.rel_frobenius(gemm_nn(a, np.ascontiguousarray(b.T), variant='tc3xtf32'), want) < 1e-5\n"
        "print('ok')\n")
    env = dict(__import__("os").environ, MTNN_TF32_INKERNEL="1", PYTHONPATH=str(ROOT))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=str(ROOT), timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr


@pytest.mark.parametrize("shape", [(1000, 128, 512), (4096, 64, 1024), (300, 112, 2048), (2048, 16, 256)])
def test_narrow_n_tile(rng, shape):
    """n <= 128 runs the BN=128 tile (no half-empty N=256 tiles); every variant
    and both B layouts stay within the FP32 gate."""
    m, n, k = shape
    a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
    want = oracle.oracle_nt_blas(a, b)
    for v in ("tc3xf16s", "tc3xtf32"):
        assert rel_frobenius(gemm_nt(a, b, variant=v), want) < FP32_GATE
        if n % 16 == 0:
            assert rel_frobenius(gemm_nn(a, np.ascontiguousarray(b.T), variant=v), want) < FP32_GATE


class TestF16SInKernelSplit:
    """Skinny shapes split the long operand inside the GEMM (raw fp32 tile ->
    fp16 h/l in shared memory, row scales from a read-only pre-pass). The halves
    are computed by the same operations as the split pass, so with the same
    output tiling (n <= 128: both paths use the 128-wide tile and the same
    split-K) C is bit-identical to the pre-split path (knob
    f16s_inkernel_max_short = 0); otherwise only the split-K summation order
    differs."""

    KEY = "f16s_inkernel_max_short"

    def _both(self, fn, *args):
        from paper_1702_03192_b200 import _lib

        old = _lib.config_get(self.KEY)
        try:
            _lib.config_set(self.KEY, 0)
            pre = fn(*args, variant="tc3xf16s")
            _lib.config_set(self.KEY, 1 << 20)
            ink = fn(*args, variant="tc3xf16s")
        finally:
            _lib.config_set(self.KEY, old)
        return pre, ink

    @pytest.mark.parametrize("shape", [(128, 4096, 2048), (4096, 128, 2048), (100, 3000, 1000),
                                       (3000, 96, 1000), (512, 2048, 4104), (300, 1100, 520),
                                       (1, 1024, 64), (1024, 4, 8)])
    def test_bit_identical_to_presplit_and_within_gate(self, rng, shape):
        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        want = oracle.oracle_nt_blas(a, b)
        pre, ink = self._both(gemm_nt, a, b)
        self._same(pre, ink, n)
        assert rel_frobenius(ink, want) < FP32_GATE
        if n % 16 == 0:  # NN: only A (K-major) is split in-kernel
            bt = np.ascontiguousarray(b.T)
            pre, ink = self._both(gemm_nn, a, bt)
            self._same(pre, ink, n)
            assert rel_frobenius(ink, want) < FP32_GATE

    @staticmethod
    def _same(pre, ink, n):
        if n <= 128:
            assert np.array_equal(pre.view(np.uint32), ink.view(np.uint32))
        else:
            assert rel_frobenius(ink, pre) < 1e-6

    def test_dynamic_range_and_nonfinite(self, rng):
        m, n, k = 2048, 192, 776
        a = (rng.standard_normal((m, k)) * np.exp(rng.uniform(-40, 40, (m, 1)))).astype(np.float32)
        b = (rng.standard_normal((n, k)) * np.exp(rng.uniform(-20, 20, (n, 1)))).astype(np.float32)
        a[7] = 0.0
        a[11, 5] = np.nan
        a[13, 9] = np.inf
        pre, ink = self._both(gemm_nt, a, b)
        assert np.array_equal(np.isnan(pre), np.isnan(ink))
        assert np.all(ink[7] == 0.0) and np.all(np.isnan(ink[11])) and np.all(~np.isfinite(ink[13]))
        ok = np.ones(m, bool); ok[[11, 13]] = False
        want = oracle.oracle_nt_blas(a[ok], b)
        err = np.linalg.norm(ink[ok] - want, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-300)
        assert err[np.linalg.norm(want, axis=1) > 0].max() < FP32_GATE

    def test_device_and_pipelined_host_paths(self, rng):
        import torch

        m, n, k = 384, 8192, 2048   # m >= 256: the host path pipelines A/C chunks
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        dev = gemm_nt(ta, tb).cpu().numpy()
        host = gemm_nt(a, b)   # row chunks: split-K may differ from the whole call
        assert rel_frobenius(host, dev) < 1e-6
        rows = np.sort(rng.choice(m, 48, replace=False))
        assert rel_frobenius(host[rows], oracle.oracle_nt_rows(a, b, rows, np.arange(n))) < FP32_GATE


class TestBlockedHostPipeline:
    """Host-buffer NT on the FP16x3 path with a wide B streams B in row blocks
    against A's first row block (C blocks leave by 2-D copies while the next B
    block arrives), then the rest of A in row chunks. Results match the device
    path (same operand halves; only split-K order may differ) and the oracle."""

    @pytest.mark.parametrize("shape", [(2048, 4096, 1024), (128, 8192, 2048), (1000, 20000, 256),
                                       (20000, 2048, 256), (10000, 9000, 1024)])
    def test_matches_device_and_oracle(self, rng, shape):
        import torch

        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        host = gemm_nt(a, b)
        dev = gemm_nt(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
        assert rel_frobenius(host, dev) < 1e-6
        rows = np.unique(np.concatenate([[0, m - 1], rng.choice(m, 40, replace=False)]))
        cols = np.unique(np.concatenate([[0, n - 1], rng.choice(n, 300, replace=False)]))
        want = oracle.oracle_nt_rows(a, b, rows, cols)
        assert rel_frobenius(host[np.ix_(rows, cols)], want) < FP32_GATE


@pytest.mark.parametrize("shape", [(1024, 10, 4096), (300, 6, 776), (2048, 130, 512), (128, 1023, 2048)])
def test_output_rows_not_tma_storable(rng, shape):
    """n % 4 != 0 (e.g. the FCN's 10-class layer): the tensor-core path computes
    into a row-padded buffer and copies the n columns out; host and device
    entry points agree with the oracle."""
    import torch

    m, n, k = shape
    a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
    want = oracle.oracle_nt_blas(a, b)
    for v in ("auto", "tc3xf16s", "tc3xtf32"):
        got = gemm_nt(a, b, variant=v)
        assert got.shape == (m, n) and rel_frobenius(got, want) < FP32_GATE
    dev = gemm_nt(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    assert rel_frobenius(dev, want) < FP32_GATE
    assert rel_frobenius(gemm_tnn(a, b), want) < FP32_GATE


class TestCtaPairTiles:
    """NT problems with >= 74 256x256 tiles run on CTA pairs (tcgen05
    cta_group::2: M = 256 MMAs, each CTA loading half of B). Each output element
    sees the same MMAs in the same order as on the single-CTA 128x256 tile, so
    with the same split-K the results are bit-identical; knob tc_pair = 2 forces
    the pair kernel on small shapes (ragged m and n, odd m-tile counts, split-K)."""

    @pytest.mark.parametrize("shape", [(256, 256, 64), (300, 520, 136), (1000, 900, 2048),
                                       (640, 4096, 8192), (2560, 2048, 1024), (384, 400, 96)])
    def test_pair_matches_single(self, rng, shape):
        import torch

        from paper_1702_03192_b200 import _lib

        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        want = oracle.oracle_nt_blas(a, b)
        old = _lib.config_get("tc_pair")
        try:
            for v in ("tc3xf16s", "tc3xtf32"):
                _lib.config_set("tc_pair", 0)
                single = gemm_nt(ta, tb, variant=v).cpu().numpy()
                _lib.config_set("tc_pair", 2)
                pair = gemm_nt(ta, tb, variant=v).cpu().numpy()
                assert rel_frobenius(pair, want) < FP32_GATE
                assert rel_frobenius(pair, single) < 1e-6
                if n % 16 == 0:  # NN: B^T MN-major, each CTA loading half its columns
                    tbt = tb.t().contiguous()
                    _lib.config_set("tc_pair", 0)
                    single = gemm_nn(ta, tbt, variant=v).cpu().numpy()
                    _lib.config_set("tc_pair", 2)
                    pair = gemm_nn(ta, tbt, variant=v).cpu().numpy()
                    assert rel_frobenius(pair, want) < FP32_GATE
                    assert rel_frobenius(pair, single) < 1e-6
        finally:
            _lib.config_set("tc_pair", old)


class TestEdgeCases:
    """Edge cases across the kernel families: degenerate and ragged dimensions,
    unaligned (offset) device views that TMA cannot take, non-finite inputs on
    the CTA-pair path, long k with tiny outputs (deep split-K)."""

    @pytest.mark.parametrize("shape", [(1, 1, 1), (1, 4096, 8), (4096, 1, 8), (7, 9, 1),
                                       (513, 257, 3), (130, 130, 130), (1, 1, 65536)])
    def test_degenerate_and_odd(self, rng, shape):
        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        want = oracle.oracle_nt_blas(a, b)
        for v in VARIANTS:
            try:
                got = gemm_nt(a, b, variant=v)
            except RuntimeError:
                assert v in ("tc3xf16s", "tc3xtf32")  # explicit TC variant on an ineligible shape
                continue
            assert got.shape == (m, n)
            assert rel_frobenius(got, want) < FP32_GATE, v
            assert rel_frobenius(gemm_tnn(a, b), want) < FP32_GATE

    def test_unaligned_device_views(self, rng):
        import torch

        m, n, k = 300, 200, 264
        a, b = random_matrix(rng, m, k + 1), random_matrix(rng, n, k + 1)
        ta = torch.from_numpy(a).cuda()[:, 1:]   # 4-byte offset rows: not TMA-aligned
        tb = torch.from_numpy(b).cuda()[:, 1:]
        want = oracle.oracle_nt_blas(np.ascontiguousarray(a[:, 1:]), np.ascontiguousarray(b[:, 1:]))
        got = gemm_nt(ta.contiguous(), tb.contiguous()).cpu().numpy()
        assert rel_frobenius(got, want) < FP32_GATE
        from paper_1702_03192_b200 import _lib
        c = torch.empty(m * n + 1, device="cuda")[1:].view(m, n)  # unaligned C base
        ac, bc = ta.contiguous(), tb.contiguous()
        _lib.check(_lib.lib.mtnn_gemm_nt(ac.data_ptr(), bc.data_ptr(), c.data_ptr(), m, n, k, 0,
                                         torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert rel_frobenius(c.cpu().numpy(), want) < FP32_GATE

    def test_nonfinite_on_pair_tiles(self, rng):
        import torch

        from paper_1702_03192_b200 import _lib

        m, n, k = 768, 512, 512
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        a[3, 5] = np.nan
        b[7, 9] = np.inf
        old = _lib.config_get("tc_pair")
        try:
            _lib.config_set("tc_pair", 2)
            got = gemm_nt(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                          variant="tc3xf16s").cpu().numpy()
        finally:
            _lib.config_set("tc_pair", old)
        assert np.all(np.isnan(got[3]))
        assert np.all(~np.isfinite(got[:, 7]))
        ok_r = np.ones(m, bool); ok_r[3] = False
        ok_c = np.ones(n, bool); ok_c[7] = False
        want = oracle.oracle_nt_blas(a[ok_r], b[ok_c])
        assert rel_frobenius(got[np.ix_(ok_r, ok_c)], want) < FP32_GATE

    @pytest.mark.parametrize("shape", [(128, 128, 262144), (256, 384, 100000)])
    def test_long_k_small_output(self, rng, shape):
        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        want = oracle.oracle_nt_blas(a, b)
        for v in ("auto", "tc3xf16s"):
            assert rel_frobenius(gemm_nt(a, b, variant=v), want) < FP32_GATE


@pytest.mark.parametrize("shape", [(4096, 4098, 1024), (2050, 8190, 512)])
def test_pair_tiles_with_padded_output(rng, shape):
    """n % 4 != 0 on a problem large enough for CTA pairs: the pair kernel writes
    the row-padded C (ldc = n rounded up), the n columns are copied out."""
    m, n, k = shape
    a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
    got = gemm_nt(a, b)
    rows = np.unique(np.r_[0, m - 1, rng.choice(m, 60, replace=False)])
    cols = np.unique(np.r_[0, n - 1, rng.choice(n, 200, replace=False)])
    assert rel_frobenius(got[np.ix_(rows, cols)], oracle.oracle_nt_rows(a, b, rows, cols)) < FP32_GATE


@pytest.mark.parametrize("path", ["nt", "nn", "tnn"])
def test_host_pipeline_with_inkernel_split_of_a(rng, path):
    """Host-buffer call on the B-first pipeline (k > 4096) whose shape splits A
    in-kernel (n <= 256, m >= 1024): every A row chunk gets its own row scales."""
    m, n, k = 4096, 208, 8192
    a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
    if path == "nt":
        got = gemm_nt(a, b)
    elif path == "nn":
        got = gemm_nn(a, np.ascontiguousarray(b.T))
    else:
        got = gemm_tnn(a, b)
    rows = np.sort(rng.choice(m, 64, replace=False))
    assert rel_frobenius(got[rows], oracle.oracle_nt_rows(a, b, rows, np.arange(n))) < FP32_GATE


def test_random_shape_fuzz(rng):
    """60 random shapes (1..2600 per dimension, biased toward odd sizes and the
    path boundaries: 128/256/1024 short sides, k near multiples of 8/32) through
    every entry point (host NT / NN / TNN, device NT) and variant, against the
    float64 oracle on sampled rows."""
    import torch

    picks = [1, 2, 3, 5, 8, 16, 31, 64, 127, 128, 129, 200, 255, 256, 257, 500, 512, 513,
             1000, 1023, 1024, 1025, 2047, 2600]
    for _ in range(60):
        m, n, k = (int(rng.choice(picks)) if rng.random() < 0.6 else int(rng.integers(1, 2600))
                   for _ in range(3))
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        rows = np.unique(rng.choice(m, min(m, 24), replace=False))
        want = oracle.oracle_nt_rows(a, b, rows, np.arange(n))
        for v in VARIANTS:
            try:
                got = gemm_nt(a, b, variant=v)
            except RuntimeError:
                assert v in ("tc3xf16s", "tc3xtf32"), (m, n, k, v)
                continue
            assert rel_frobenius(got[rows], want) < FP32_GATE, (m, n, k, v)
        assert rel_frobenius(gemm_tnn(a, b)[rows], want) < FP32_GATE, (m, n, k, "tnn")
        assert rel_frobenius(gemm_nn(a, np.ascontiguousarray(b.T))[rows], want) < FP32_GATE, (m, n, k, "nn")
        dev = gemm_nt(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
        assert rel_frobenius(dev[rows], want) < FP32_GATE, (m, n, k, "device")


@pytest.mark.parametrize("k", [8, 96, 256, 264, 512, 520, 1024, 1032, 2048, 2056, 4096, 4104,
                               8192, 8200, 16384, 16392, 40960, 41000])
@pytest.mark.parametrize("n", [384, 200])
def test_row_split_every_branch(rng, k, n):
    """Every row-split kernel (looped / register warp-per-row / register
    CTA-per-row / smem-staged / past the smem limit) picked by k, for pre-split
    operands (n = 384) and row-scale-only jobs of the in-kernel split (n = 200),
    on rows whose magnitudes span 2^-40..2^40: each output row within the gate
    relative to its own norm; a NaN at a row's last element poisons exactly
    that row."""
    m = 384
    a = random_matrix(rng, m, k) * np.exp2(rng.integers(-40, 41, m)).astype(np.float32)[:, None]
    b = random_matrix(rng, n, k) * np.exp2(rng.integers(-40, 41, n)).astype(np.float32)[:, None]
    a[5, k - 1] = np.nan
    got = gemm_nt(a, b, variant="tc3xf16s")
    assert np.all(np.isnan(got[5]))
    ok = np.arange(m) != 5
    want = oracle.oracle_nt_blas(a[ok], b)
    g = got[ok]
    err = np.linalg.norm(g - want, axis=1) / np.linalg.norm(want, axis=1)
    assert err.max() < FP32_GATE, (k, n, float(err.max()))


@pytest.mark.parametrize("k", [8, 104, 128, 256, 264, 1024, 1032, 2048, 2056, 4096, 4104, 8192, 8200,
                               16384])
@pytest.mark.parametrize("n", [208, 384, 1072])
def test_col_split_every_branch(rng, k, n):
    """NN (MN-major B^T) column split — one scale per (256-row chunk, column) —
    at chunk-ragged k (k % 256 != 0, k < 256), ragged 32-column blocks
    (n % 32 != 0), columns whose magnitudes span 2^-40..2^40 AND change by up to
    2^+-20 from one k-row to the next (every chunk gets its own scale), and a
    NaN in the last row of one column poisoning exactly that output column."""
    m = 384
    a = random_matrix(rng, m, k) * np.exp2(rng.integers(-40, 41, m)).astype(np.float32)[:, None]
    bt = (random_matrix(rng, k, n) * np.exp2(rng.integers(-40, 41, n)).astype(np.float32)[None, :]
          * np.exp2(rng.integers(-20, 21, k)).astype(np.float32)[:, None])
    bt[k - 1, 7] = np.nan
    got = gemm_nn(a, bt, variant="tc3xf16s")
    assert np.all(np.isnan(got[:, 7]))
    ok = np.arange(n) != 7
    want = np.asarray(a, np.float64) @ np.asarray(bt[:, ok], np.float64)
    g = got[:, ok]
    err = np.linalg.norm(g - want, axis=0) / np.linalg.norm(want, axis=0)
    assert err.max() < FP32_GATE, (k, n, float(err.max()))


@pytest.mark.parametrize("m,n,k", [(256, 256, 4104), (128, 512, 8200), (256, 256, 16384),
                                   (2304, 2304, 1000), (2304, 2304, 4360), (512, 4096, 2056)])
def test_nn_chunk_scales_with_split_k_and_pairs(rng, m, n, k):
    """MN-major chunk scales through split-K (k-splits start on 256-row chunk
    boundaries) and the CTA-pair kernel (>= 74 pair tiles), with B^T rows whose
    magnitudes change per k-row; NN, TNN and the host entry point agree with
    float64 and NN == TNN bit for bit (same kernels on the same B^T)."""
    k -= k % 8
    a = random_matrix(rng, m, k)
    bt = random_matrix(rng, k, n) * np.exp2(rng.integers(-12, 13, k)).astype(np.float32)[:, None]
    want = np.asarray(a, np.float64) @ np.asarray(bt, np.float64)
    nn = gemm_nn(a, bt, variant="tc3xf16s")
    tnn = gemm_tnn(a, np.ascontiguousarray(bt.T), variant="tc3xf16s")
    assert rel_frobenius(nn, want) < FP32_GATE
    assert np.array_equal(nn, tnn)
    import torch

    dev = kernels.gemm_nn(torch.from_numpy(a).cuda(), torch.from_numpy(bt).cuda(),
                          variant="tc3xf16s").cpu().numpy()
    assert np.array_equal(dev, nn)


@pytest.mark.parametrize("shape", [(1024, 10, 4096), (10, 4096, 1024), (1, 1, 4), (13, 13, 4096),
                                   (7, 300, 1000), (3000, 16, 3200), (16, 5000, 12800),
                                   (20000, 3, 64), (2, 70000, 8)])
def test_skinny_outputs(rng, shape):
    """Outputs with a side <= 16 (the FCN's 10-class layer, GEMV-like products):
    the shared-memory SIMT kernel (or, past its 200 KiB short operand, the tile
    kernels) through the device and host entry points, against the oracle; NaN
    in a long-operand row poisons exactly that output line."""
    import torch

    m, n, k = shape
    a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
    want = oracle.oracle_nt_blas(a, b)
    assert rel_frobenius(gemm_nt(a, b), want) < FP32_GATE
    dev = gemm_nt(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    assert rel_frobenius(dev, want) < FP32_GATE
    if m >= n:
        a[m // 2, k - 1] = np.nan
        got = gemm_nt(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
        assert np.all(np.isnan(got[m // 2]))
        assert np.isfinite(np.delete(got, m // 2, axis=0)).all()
    else:
        b[n // 2, k - 1] = np.nan
        got = gemm_nt(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
        assert np.all(np.isnan(got[:, n // 2]))
        assert np.isfinite(np.delete(got, n // 2, axis=1)).all()


@pytest.mark.parametrize("shape", [(1024, 4096, 10), (1, 1, 1), (7, 13, 3), (513, 1001, 16),
                                   (4096, 10, 12), (3, 70000, 5)])
def test_short_k(rng, shape):
    """k <= 16 (the FCN's backward NN through the 10-class layer) through NT,
    NN, TNN, host and device entry points."""
    import torch

    m, n, k = shape
    a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
    want = oracle.oracle_nt_blas(a, b)
    assert rel_frobenius(gemm_nt(a, b), want) < FP32_GATE
    assert rel_frobenius(gemm_nt(a, b, variant="ffma"), want) < FP32_GATE
    bt = np.ascontiguousarray(b.T)
    assert rel_frobenius(gemm_nn(a, bt), want) < FP32_GATE
    assert rel_frobenius(gemm_tnn(a, b), want) < FP32_GATE
    dev = kernels.gemm_nn(torch.from_numpy(a).cuda(), torch.from_numpy(bt).cuda()).cpu().numpy()
    assert rel_frobenius(dev, want) < FP32_GATE


@pytest.mark.parametrize("switch", ["MTNN_PDL=0", "MTNN_SPLIT_CTAREG=0", "MTNN_SKINNY=0",
                                    "MTNN_PAIR_MAXK=4096"])
def test_env_switches_keep_results(tmp_path, switch):
    """Every A/B environment switch (read once per process) keeps results within
    the FP32 gate on the shapes it affects, and the switches that change only
    scheduling or the split kernel (not the arithmetic) keep them bit-identical
    to the default process."""
    import subprocess
    import sys

    from conftest import ROOT

    code = (
        "import sys, numpy as np, oracle\n"
        "from paper_1702_03192_b200 import gemm_nt, gemm_nn\n"
        "rng = np.random.default_rng(11)\n"
        "outs = []\n"
        "for m, n, k in ((1024, 10, 4096), (384, 384, 4104), (512, 1072, 3000), (2048, 2048, 8192)):\n"
        "    k -= k % 8\n"
        "    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)\n"
        "    b = rng.uniform(-1, 1, (n, k)).astype(np.float32)\n"
        "    want = oracle.oracle_nt_blas(a, b)\n"
        "    c1 = gemm_nt(a, b)\n"
        "    c2 = gemm_nn(a, np.ascontiguousarray(b.T)) if n % 16 == 0 else c1\n"
        "    assert oracle.rel_frobenius(c1, want) < 1e-5 and oracle.rel_frobenius(c2, want) < 1e-5\n"
        "    outs += [c1, c2]\n"
        "np.savez(sys.argv[1], *outs)\n"
        "print('ok')\n")
    base = dict(__import__("os").environ, PYTHONPATH=str(ROOT))
    key, val = switch.split("=")
    res = {}
    for name, env in (("default", base), ("switch", dict(base, **{key: val}))):
        path = tmp_path / f"{name}.npz"
        out = subprocess.run([sys.executable, "-c", code, str(path)], capture_output=True,
                             text=True, env=env, cwd=str(ROOT), timeout=300)
        assert out.returncode == 0 and "ok" in out.stdout, out.stderr
        res[name] = np.load(path)
    if key in ("MTNN_PDL", "MTNN_SPLIT_CTAREG"):
        for f in res["default"].files:
            assert np.array_equal(res["default"][f], res["switch"][f]), (switch, f)


class TestDeviceValidation:
    """device.* is called directly by sweep/evaluate/tools: shape and device
    errors must raise before any pointer reaches the C ABI (a bad k would read
    out of bounds and poison the context)."""

    def test_inner_dimension_mismatch(self):
        import torch

        from paper_1702_03192_b200 import device

        a = torch.zeros(64, 32, device="cuda")
        b = torch.zeros(48, 40, device="cuda")
        with pytest.raises(ValueError, match="share k"):
            device.gemm_nt(a, b)
        with pytest.raises(ValueError, match="share k"):
            device.gemm_tnn(a, b)
        with pytest.raises(ValueError, match="share k"):
            device.gemm_nn(a, torch.zeros(40, 48, device="cuda"))
        with pytest.raises(ValueError, match="shape"):
            device.gemm_nt(a, torch.zeros(48, 32, device="cuda"), out=torch.zeros(64, 47, device="cuda"))
        torch.cuda.synchronize()  # the context is still healthy
        c = device.gemm_nt(a, torch.ones(48, 32, device="cuda"))
        assert float(c.abs().sum()) == 0.0

    def test_host_and_device_mix_rejected(self):
        import torch

        a = torch.zeros(8, 8, device="cuda")
        with pytest.raises(TypeError):
            gemm_nt(a, np.zeros((8, 8), np.float32))


def test_stream_gate_holds_until_released():
    """mtnn_gate (bench.py's window gate) holds the stream until the host writes
    the value into the pinned flag; a pageable flag is rejected."""
    import ctypes
    import time

    import torch

    from paper_1702_03192_b200 import _lib

    flag = torch.zeros(1, dtype=torch.int32).pin_memory()
    s = torch.cuda.current_stream()
    # (allocate and load the kernel first: a first-use allocation or a lazy
    # module load behind a held gate synchronises, returning only once the
    # gate's 1 s bound expires — bench.py gates only after its warm-up steps)
    x = torch.ones(4, device="cuda")
    y = torch.empty_like(x)
    torch.mul(x, 2, out=y)
    torch.cuda.synchronize()
    _lib.check(_lib.lib.mtnn_gate(flag.data_ptr(), 1, s.cuda_stream))
    done = torch.cuda.Event()
    torch.mul(x, 2, out=y)
    done.record()
    time.sleep(0.05)
    assert not done.query()  # held at the gate
    flag.numpy()[0] = 1
    done.synchronize()
    assert torch.equal(y.cpu(), torch.full((4,), 2.0))
    pageable = (ctypes.c_int32 * 1)()
    with pytest.raises(ValueError, match="pinned"):
        _lib.check(_lib.lib.mtnn_gate(ctypes.addressof(pageable), 1, s.cuda_stream))


def test_gated_window_excludes_host_stalls():
    """bench.py's timing method: a window opened behind the gate and released
    after the call is enqueued holds device time only, even if the host stalls
    20 ms while enqueueing."""
    import time

    import torch

    from paper_1702_03192_b200 import _lib, device

    a = torch.rand(512, 512, device="cuda")
    b = torch.rand(512, 512, device="cuda")
    device.gemm_nt(a, b)  # load kernels, grow pools
    flag = torch.zeros(1, dtype=torch.int32).pin_memory()
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()
    _lib.check(_lib.lib.mtnn_gate(flag.data_ptr(), 1, s.cuda_stream))
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    time.sleep(0.02)  # a host stall inside the window
    device.gemm_nt(a, b)
    t1.record()
    flag.numpy()[0] = 1
    torch.cuda.synchronize()
    assert t0.elapsed_time(t1) < 5.0  # ms: the GEMM, not the 20 ms stall


class TestGemvClassKernels:
    """GEMV-class products on the SIMT kernels: the staged skinny NT (output side
    <= 16: the long operand's rows bulk-copied into shared memory, the short
    operand in registers) and the small-k NN (k <= 16: outer-product sum bound by
    writing C) — against float64, through the dispatcher's auto variant, on
    both skinny orientations and one- and multi-step k."""

    @pytest.mark.parametrize("shape", [(1024, 10, 4096), (10, 4096, 1024), (2000, 3, 2048),
                                       (7, 1500, 16384), (4096, 16, 512), (333, 1, 1028),
                                       (1, 5000, 64)])
    def test_skinny_nt(self, rng, shape):
        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        want = a.astype(np.float64) @ b.astype(np.float64).T
        got = gemm_nt(a, b)
        assert rel_frobenius(got, want) < FP32_GATE
        assert np.array_equal(got, gemm_nt(a, b))  # fixed summation order

    # streaming skinny NT (<= 10 short rows, long operand <= 32 MB): one k-range
    # (no cluster), clusters of 2 / 4 / 8 CTAs along k, more ranges than a
    # cluster (second-pass fold), ragged k-ranges and row blocks, both
    # orientations, short sides 1..10
    @pytest.mark.parametrize("shape", [(4096, 10, 1024), (10, 4096, 1024), (1024, 10, 4096),
                                       (2000, 7, 2052), (3, 777, 8192), (256, 10, 16384),
                                       (100, 9, 9000), (1, 1, 4), (4099, 2, 1000), (5, 64, 20000)])
    def test_streaming_skinny_nt(self, rng, shape):
        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        want = a.astype(np.float64) @ b.astype(np.float64).T
        got = gemm_nt(a, b)
        assert rel_frobenius(got, want) < FP32_GATE
        assert np.array_equal(got, gemm_nt(a, b))  # fixed fold order

    @pytest.mark.parametrize("shape", [(1024, 4096, 10), (33, 100, 16), (5, 8, 1), (300, 1028, 7),
                                       (4097, 260, 4), (64, 4096, 13)])
    def test_smallk_nn_and_tnn(self, rng, shape):
        m, n, k = shape
        a, b = random_matrix(rng, m, k), random_matrix(rng, n, k)
        want = a.astype(np.float64) @ b.astype(np.float64).T
        got = gemm_nn(a, np.ascontiguousarray(b.T))
        assert rel_frobenius(got, want) < FP32_GATE
        assert rel_frobenius(gemm_tnn(a, b), want) < FP32_GATE
        # k = 1: every output is one product, exact
        if k == 1:
            assert np.array_equal(got, (a @ b.T).astype(np.float32))

