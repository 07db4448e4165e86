#!/bin/bash
# Conformance: run the REFERENCE's own unit tests (read-only, from
# /root/reference -- only present in the build container) against the
# drop-in through the import alias of INTEGRATION.md.  Nothing is copied.
#   tools/run_reference_tests.sh [test files...]   (default: mesh, quadrature, kernels)
set -e
REF=${HVBEM_REF_TESTS:-/root/reference/pkg/tests}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
ALIAS=$(mktemp -d)
cat > "$ALIAS/sitecustomize.py" <<PY
import importlib, sys
sys.path.insert(0, "$ROOT")
sys.modules["hvbem"] = importlib.import_module("paper_2003_12663_b200")
for sub in ("mesh", "quadrature", "kernels", "assembly", "solver", "postprocess", "fixtures", "config", "cli"):
    sys.modules[f"hvbem.{sub}"] = importlib.import_module(f"paper_2003_12663_b200.{sub}")
PY
files=("$@")
[ ${#files[@]} -eq 0 ] && files=("$REF/test_mesh.py" "$REF/test_quadrature.py" "$REF/test_kernels.py")
cd "$ALIAS"
PYTHONDONTWRITEBYTECODE=1 PYTHONPATH="$ALIAS" python -m pytest -p no:cacheprovider -q "${files[@]}"
