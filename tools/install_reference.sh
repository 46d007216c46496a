#!/bin/bash
# Install the UNMODIFIED reference into baseline/_ref (git-ignored; travels to the
# GPU box with gpurun) from a /tmp copy of /root/reference/pkg, plus its own test
# suite (baseline/_ref/tests) so tests/test_reference_suite_gpu.py can run it
# against the B200 backend where /root/reference does not exist.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/mtnn_ref_src baseline/_ref
cp -r /root/reference/pkg /tmp/mtnn_ref_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/mtnn_ref_src --no-deps
cp -r /root/reference/pkg/tests baseline/_ref/tests
find baseline/_ref -name __pycache__ -prune -exec rm -rf {} +
echo "installed: $(ls baseline/_ref)"
