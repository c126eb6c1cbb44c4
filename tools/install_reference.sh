#!/bin/bash
# Stage the reference for the bench's reference arm and the reference-suite
# run (run HERE, where /root/reference exists; baseline/_ref is git-ignored
# but travels to the GPU box with the gpurun snapshot):
#   baseline/_ref/lpqt   the unmodified reference package (pip --target)
#   baseline/_ref/tests  the reference's own tests (pkg/tests), run against
#                        the drop-in by tests/test_reference_suite.py
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/lpqt_refsrc baseline/_ref
cp -r /root/reference/pkg /tmp/lpqt_refsrc
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/lpqt_refsrc
cp -r /root/reference/pkg/tests baseline/_ref/tests
find baseline/_ref -name __pycache__ -prune -exec rm -rf {} +
echo "reference staged in baseline/_ref"
