#!/bin/sh
# Install the UNMODIFIED reference (package `ncstream`, pure Python) into baseline/_ref, the one
# offline install the task allows.  baseline/_ref is git-ignored but travels to the GPU box with
# the gpurun snapshot, where /root/reference does not exist.  It provides:
#   * the reference arm of bench.py (`--impl reference` times ncstream's own
#     multi_head_attention_array on the host cores),
#   * ncstream's exception classes / DenseTensor for the drop-in boundary (_reftypes.py),
#   * the reference's own test files (copied unmodified to baseline/_ref/ncstream_tests), run
#     against the GPU path by tests/test_reference_suite.py.
# matplotlib (plots.py only, imported lazily) is absent offline: --no-deps.
set -e
cd "$(dirname "$0")/.."
SRC=${NCSTREAM_SRC:-/root/reference/pkg}
rm -rf /tmp/ncstream_src baseline/_ref
cp -r "$SRC" /tmp/ncstream_src   # the source tree is read-only; setuptools writes build files
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/ncstream_src
cp -r "$SRC/tests" baseline/_ref/ncstream_tests
echo "installed ncstream into baseline/_ref"
