"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container only (it imports the read-only reference package
from /root/reference/pkg/src; that tree does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Outputs (committed, small):
  kernels.npz    operands + reference outputs of gemm_nt / gemm_tnn / gemm_nn /
                 transpose_oop (numba backend, float32) and the float64
                 oracle_nt, over the shapes the reference tests use
                 (test_kernels.py:28-175, test_acceptance.py:68-101)
  models/*.json  GBDT models trained by the reference's fit_gbdt, serialized by
                 its serialize_model (gbdt.py:388-405)
  selector.npz   per model: packed arrays (selector._pack_trees), feature
                 vectors, reference predict_raw / predict labels, and
                 Dispatcher.select decisions under given free-memory values
  operands.npz   bench.make_operands outputs (bench.py:104-114)
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_golden")
    sys.path.insert(0, str(REF))
    import mtnn
    from mtnn import bench, gbdt, selector
    from mtnn.kernels import _numba_impl
    from mtnn.platform import PlatformFeatures

    assert mtnn.active_backend() == "numba", "golden vectors must come from the numba backend"
    rng = np.random.default_rng(1234)

    def rmat(r, c):
        return rng.uniform(-1.0, 1.0, (r, c)).astype(np.float32)

    def oracle_nt(a, b):
        return a.astype(np.float64) @ b.astype(np.float64).T

    # ------------------------------------------------------------- kernels
    shapes = [(1, 1, 1), (1, 2, 3), (2, 3, 5), (3, 3, 3), (5, 8, 17), (17, 5, 2),
              (8, 17, 8), (37, 53, 29), (64, 64, 64), (130, 130, 130), (33, 1, 64),
              (1, 47, 64)]
    for _ in range(12):
        shapes.append(tuple(int(v) for v in rng.integers(1, 65, size=3)))
    data = {"shapes": np.array(shapes, dtype=np.int64)}
    for i, (m, n, k) in enumerate(shapes):
        a, b = rmat(m, k), rmat(n, k)
        b_kn = np.ascontiguousarray(b.T)
        data[f"a{i}"] = a
        data[f"b{i}"] = b
        data[f"nt{i}"] = _numba_impl.gemm_nt(a, b)
        data[f"tnn{i}"] = _numba_impl.gemm_tnn(a, b, 128, 32)
        data[f"nn{i}"] = _numba_impl.gemm_nn(a, b_kn, 64)
        data[f"t{i}"] = _numba_impl.transpose_oop(b, 32)
        data[f"f64_{i}"] = oracle_nt(a, b)
    # identities and KATs (test_kernels.py:28-40, 83-89, 113-116, 151-153)
    data["kat_nn"] = _numba_impl.gemm_nn(np.array([[2.0]], np.float32), np.array([[3.0]], np.float32), 128)
    data["kat_nt"] = _numba_impl.gemm_nt(np.array([[1.0, 2.0]], np.float32), np.array([[3.0, 4.0]], np.float32))
    data["kat_t_in"] = np.array([[1, 2, 3], [4, 5, 6]], np.float32)
    data["kat_t_out"] = _numba_impl.transpose_oop(data["kat_t_in"], 32)
    data["kat_tnn"] = _numba_impl.gemm_tnn(np.array([[2.0]], np.float32), np.array([[-3.0]], np.float32), 128, 32)
    ident_a = rmat(130, 130)
    data["ident_a"] = ident_a
    data["ident_nn"] = _numba_impl.gemm_nn(ident_a, np.eye(130, dtype=np.float32), 64)
    data["ident_nt"] = _numba_impl.gemm_nt(ident_a[:3, :3].copy(), np.eye(3, dtype=np.float32))
    # transpose of raw bit patterns (NaN payloads, -0.0, infinities, subnormals)
    bits = rng.integers(0, 2**32, size=(37, 65), dtype=np.uint64).astype(np.uint32)
    bits[0, :4] = [0x80000000, 0x7FC00001, 0xFF800000, 0x00000001]
    data["bits_in"] = bits
    data["bits_out"] = _numba_impl.transpose_oop(bits.view(np.float32), 32).view(np.uint32)
    np.savez_compressed(OUT / "kernels.npz", **data)

    # ------------------------------------------------------------- models
    models_dir = OUT / "models"
    models_dir.mkdir(exist_ok=True)
    plat_a = PlatformFeatures(gm=8.0, sm=20.0, cc=1607.0, mbw=256.0, l2c=2048.0)
    models = {}

    # (1) the selector tests' size rule (test_selector.py:21-35)
    n = 300
    x = np.column_stack([np.full(n, 8.0), np.full(n, 20.0), np.full(n, 1607.0),
                         np.full(n, 256.0), np.full(n, 2048.0),
                         rng.integers(1, 1025, n), rng.integers(1, 1025, n),
                         rng.integers(1, 1025, n)]).astype(np.float64)
    y = np.where(x[:, 5] * x[:, 6] * x[:, 7] < 2**24, 1, -1)
    models["size_rule"] = gbdt.fit_gbdt(x, y)
    # (2) constant models (test_selector.py:38-40)
    xc = rng.uniform(size=(20, 8))
    models["const_pos"] = gbdt.fit_gbdt(xc, np.full(20, 1))
    models["const_neg"] = gbdt.fit_gbdt(xc, np.full(20, -1))
    # (3) the reference pipeline on its deterministic fixture timings
    #     (bench.synthetic_timings -> label_records -> fit_gbdt), grid 2^5..2^11
    injected = {tuple(s): bench.synthetic_timings(s) for s in bench.grid_shapes(range(5, 12))}
    records = bench.sweep_grid(range(5, 12), plat_a, injected=injected)
    xs, ys = bench.samples_to_arrays(bench.label_records(records, plat_a))
    models["fixture"] = gbdt.fit_gbdt(xs, ys)
    models["fixture_squared"] = gbdt.fit_gbdt(xs, ys, gbdt.GbdtParams(max_depth=4, n_estimators=3,
                                                                     eta=0.3, objective="squared"))
    # (4) float-precision round trip (test_gbdt.py:317-324)
    leaf = lambda w: gbdt.TreeNode(weight=w)
    tree = gbdt.TreeNode(feature=5, threshold=1.0 / 3.0,
                         left=leaf(-1e-17),
                         right=gbdt.TreeNode(feature=7, threshold=np.pi, left=leaf(0.1), right=leaf(-0.0)))
    models["precision"] = gbdt.GbdtModel(trees=(tree,), params=gbdt.GbdtParams(n_estimators=2),
                                         base_score=0.0, n_features=8)
    models["empty"] = gbdt.GbdtModel(trees=(), params=gbdt.GbdtParams(), n_features=8)

    sel = {}
    for name, model in models.items():
        (models_dir / f"{name}.json").write_text(gbdt.serialize_model(model))
        feat, thresh, left, right, leaf_w = selector._pack_trees(model)
        sel[f"{name}/feat"] = feat
        sel[f"{name}/thresh"] = thresh
        sel[f"{name}/left"] = left
        sel[f"{name}/right"] = right
        sel[f"{name}/leaf"] = leaf_w
        # feature vectors: random shapes, sweep-grid shapes, and exact thresholds
        shapes_s = [tuple(int(v) for v in rng.integers(1, 4097, 3)) for _ in range(600)]
        shapes_s += [tuple(int(2 ** e) for e in t) for t in rng.integers(5, 15, size=(200, 3))]
        ths = [t for t in np.unique(thresh[feat >= 5])] if (feat >= 5).any() else []
        for t in ths[:50]:
            v = float(t)
            shapes_s.append((max(1, int(np.floor(v))), max(1, int(np.ceil(v))), max(1, int(round(v)))))
        fv = np.array([list(plat_a.as_tuple()) + [float(s) for s in sh] for sh in shapes_s])
        if name == "precision":
            # hit the exact thresholds too (float features)
            fv = np.vstack([fv, np.array([[8, 20, 1607, 256, 2048, 1.0 / 3.0, 1, np.pi],
                                          [8, 20, 1607, 256, 2048, 0.3333, 1, 3.0]])])
        raws = np.array([gbdt.predict_raw(model, v) for v in fv])
        labels = np.array([gbdt.predict(model, v) for v in fv])
        sel[f"{name}/x"] = fv
        sel[f"{name}/raw"] = raws
        sel[f"{name}/label"] = labels
        # Dispatcher.select under ample and tight free memory
        disp = selector.Dispatcher(model, plat_a)
        free = rng.integers(0, 4 * 4096 * 4096, size=len(shapes_s))
        dec_choice, dec_reason, dec_raw = [], [], []
        for sh, fr in zip(shapes_s, free):
            d = disp.select(mtnn.ProblemShape(*sh), int(fr))
            dec_choice.append(1 if d.choice is selector.Choice.USE_TNN else 0)
            dec_reason.append(1 if d.reason is selector.Reason.MEMORY_FALLBACK else 0)
            dec_raw.append(d.raw_score)
        sel[f"{name}/shapes"] = np.array(shapes_s, dtype=np.int64)
        sel[f"{name}/free"] = free.astype(np.int64)
        sel[f"{name}/choice"] = np.array(dec_choice, dtype=np.int64)
        sel[f"{name}/reason"] = np.array(dec_reason, dtype=np.int64)
        sel[f"{name}/sel_raw"] = np.array(dec_raw, dtype=np.float64)
        sel[f"{name}/base"] = np.array([model.base_score, model.params.eta])
    sel["prefix"] = np.array(plat_a.as_tuple())
    np.savez_compressed(OUT / "selector.npz", **sel)

    # ------------------------------------------------------------- operands
    ops = {}
    for i, (shape, seed) in enumerate([((4, 5, 6), 0), ((3, 2, 7), 7), ((16, 8, 4), 123)]):
        a, b, b_kn = bench.make_operands(mtnn.ProblemShape(*shape), seed)
        ops[f"shape{i}"] = np.array(shape + (seed,))
        ops[f"a{i}"], ops[f"b{i}"], ops[f"bkn{i}"] = a, b, b_kn
    np.savez_compressed(OUT / "operands.npz", **ops)
    # ------------------------------------------------------------- evaluation layer
    from mtnn import metrics

    ev = {}
    for i, n_cases in enumerate((40, 7)):
        p = rng.uniform(1.0, 400.0, size=(n_cases, 3))
        p[::5, 2] = p[::5, 0]          # some cases equal to a branch (copied mode)
        p[1, 2] = 2.5 * p[1, 0]        # >= 2.0 histogram bucket
        cases = [metrics.EvalCase(shape=mtnn.ProblemShape(1, 1, 1), p_nt=a_, p_tnn=b_, p_mtnn=c_)
                 for a_, b_, c_ in p]
        rep = metrics.aggregate(cases, p_mtnn_mode="copied" if i else "remeasured")
        ev[f"p{i}"] = p
        ev[f"vals{i}"] = np.array([rep.mtnn_vs_nt, rep.mtnn_vs_tnn, rep.gow_avg, rep.gow_max,
                                   rep.lub_avg, rep.lub_min])
        ev[f"hist{i}"] = np.array(rep.ratio_histogram)
        (OUT / f"report{i}.txt").write_text(metrics.render_report(rep) + "\n")
    np.savez_compressed(OUT / "evaluate.npz", **ev)
    # records / samples CSV wire formats from injected (synthetic) timings
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        injected = {tuple(s): bench.synthetic_timings(s) for s in bench.grid_shapes(range(5, 8))}
        recs = bench.sweep_grid(range(5, 8), plat_a, injected=injected)
        bench.write_records_csv(f"{td}/r.csv", recs)
        bench.write_samples_csv(f"{td}/s.csv", bench.label_records(recs, plat_a))
        bench.write_timings_csv(f"{td}/t.csv", range(5, 8))
        for name in ("r", "s", "t"):
            (OUT / f"wire_{name}.csv").write_text(open(f"{td}/{name}.csv").read())

    meta = {"reference": str(REF), "backend": mtnn.active_backend(),
            "numpy": np.__version__, "models": sorted(models)}
    (OUT / "MANIFEST.json").write_text(json.dumps(meta, indent=1))
    print("wrote golden fixtures to", OUT)


if __name__ == "__main__":
    main()
