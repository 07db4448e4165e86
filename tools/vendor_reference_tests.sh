#!/bin/bash
# Vendor the reference's own test modules (hvbem 0.1.0, pkg/tests) VERBATIM
# into tests/reference_suite/ as test infrastructure: they run against the
# drop-in through the INTEGRATION.md import alias on the GPU box
# (tests/test_reference_suite.py), where /root/reference does not exist.
# MANIFEST.sha256 records the source hashes (verbatim copies, unmodified).
set -e
REF=${HVBEM_REF_TESTS:-/root/reference/pkg/tests}
DST=$(cd "$(dirname "$0")/.." && pwd)/tests/reference_suite
mkdir -p "$DST"
files="conftest.py oracles.py test_assembly.py test_solver.py test_postprocess.py test_acceptance.py test_mesh.py test_quadrature.py test_kernels.py"
: > "$DST/MANIFEST.sha256"
for f in $files; do
  cp "$REF/$f" "$DST/$f"
  (cd "$DST" && sha256sum "$f" >> MANIFEST.sha256)
done
echo "vendored: $files"
