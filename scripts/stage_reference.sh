#!/bin/sh
# Stage the UNMODIFIED reference package and its tests under baseline/_ref/ (git-ignored,
# shipped to the GPU box with the gpurun snapshot).  Used by the drop-in tests
# (tests/test_reference_unmodified_gpu.py, test_parity_gpu.py::test_shim_routes_reference_api).
set -e
cd "$(dirname "$0")/.."
SRC=${1:-/root/reference/pkg}
rm -rf baseline/_ref/megores baseline/_ref/tests
mkdir -p baseline/_ref
cp -r "$SRC/src/megores" baseline/_ref/megores
cp -r "$SRC/tests" baseline/_ref/tests
find baseline/_ref -name __pycache__ -prune -exec rm -rf {} +
echo "staged $(ls baseline/_ref/megores | wc -l) package files, $(ls baseline/_ref/tests | wc -l) test files"
