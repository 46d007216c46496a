"""The reference's OWN kernel and selector test suites
(pkg/tests/test_kernels.py, test_selector.py) run against the B200 backend:
the installed reference (baseline/_ref) with INTEGRATION.md §1-3 applied to a
copy (tests/ref_binding.py), MTNN_BACKEND=b200. Proves the drop-in boundary
from the reference side.

Deselected (they assume a CPU backend by name or a pip-installed ``mtnn`` in
a bare-PATH subprocess): test_env_flag_selects_backend,
test_invalid_env_flag_rejected, test_active_backend_reports.
"""

import os
import subprocess
import sys

import pytest

from ref_binding import REF, ROOT, bind

pytestmark = pytest.mark.gpu

DESELECT = ("test_env_flag_selects_backend", "test_invalid_env_flag_rejected",
            "test_active_backend_reports")


@pytest.mark.skipif(not (REF / "tests").is_dir(),
                    reason="baseline/_ref not installed (tools/install_reference.sh)")
@pytest.mark.parametrize("suite", ["test_kernels.py", "test_selector.py"])
def test_reference_suite_on_b200(tmp_path, suite):
    bind(tmp_path)
    env = dict(os.environ, MTNN_BACKEND="b200", NUMBA_CACHE_DIR=str(tmp_path / "numba"),
               PYTHONPATH=os.pathsep.join([str(tmp_path), str(ROOT)]))
    probe = subprocess.run([sys.executable, "-c",
                            "import mtnn, mtnn.selector as s; print(mtnn.active_backend(), "
                            "s._impl.__name__)"], env=env, capture_output=True, text=True,
                           cwd=str(tmp_path))
    assert probe.returncode == 0, probe.stderr[-2000:]
    assert probe.stdout.split() == ["b200", "mtnn.kernels._b200_impl"], probe.stdout
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          str(REF / "tests" / suite), "-k",
                          " and ".join(f"not {t}" for t in DESELECT),
                          "--rootdir", str(tmp_path)],
                         env=env, capture_output=True, text=True, cwd=str(tmp_path), timeout=1200)
    tail = out.stdout[-3000:]
    print(tail)
    assert out.returncode == 0, tail + out.stderr[-2000:]
    assert " passed" in tail and "failed" not in tail
