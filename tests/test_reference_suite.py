"""The reference's OWN test suite against the drop-in ("the
reference test suite can itself run against the drop-in (import alias) as a
conformance gate").  The modules are vendored verbatim from hvbem 0.1.0
pkg/tests (tests/reference_suite/, hashes in MANIFEST.sha256,
tools/vendor_reference_tests.sh) and run in a subprocess in which
``import hvbem`` resolves to paper_2003_12663_b200 (INTEGRATION.md alias).

Outcomes that are NOT parity failures are listed in KNOWN with the reason;
any other failure fails this test, and the pass count is printed."""

import hashlib
import os
import re
import subprocess
import sys
import tempfile

import pytest

from conftest import gpu_ok

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "tests", "reference_suite")

# test id -> why it cannot pass on the device path (not an arithmetic difference)
KNOWN = {
    "test_acceptance.py::test_criterion_8_scaling_exponent":
        "asserts the CPU reference's O(N^2) time-vs-N exponent in [1.7, 2.3] over a 642/2562/10242 ladder; the "
        "device assembly of these sizes takes milliseconds and is launch-bound, so its exponent is far lower",
    "test_acceptance.py::test_criterion_8_parallel_speedup":
        "asserts a >2x speedup from workers=8 over workers=1; `workers` is accepted for signature compatibility "
        "but the device path does not use host threads (SURVEY 8b Threading)",
    "test_quadrature.py::test_subdivide_always_partitions":
        "hypothesis property test; at the example it can find, (0.5, 8.85e-12), the REFERENCE itself fails the "
        "property and the drop-in returns the reference's subdivision (VERDICT r1); passes when not drawn",
}

ALIAS = """import importlib, sys
sys.path.insert(0, {root!r})
sys.modules["hvbem"] = importlib.import_module("paper_2003_12663_b200")
for sub in ("mesh", "quadrature", "kernels", "assembly", "solver", "postprocess", "fixtures", "config", "cli"):
    sys.modules[f"hvbem.{{sub}}"] = importlib.import_module(f"paper_2003_12663_b200.{{sub}}")
"""


def test_vendored_suite_is_verbatim():
    for line in open(os.path.join(SUITE, "MANIFEST.sha256")):
        digest, name = line.split()
        assert hashlib.sha256(open(os.path.join(SUITE, name), "rb").read()).hexdigest() == digest, name


def _run(files, timeout):
    with tempfile.TemporaryDirectory() as tmp:
        with open(os.path.join(tmp, "sitecustomize.py"), "w") as fh:
            fh.write(ALIAS.format(root=ROOT))
        env = dict(os.environ, PYTHONPATH=tmp, PYTHONDONTWRITEBYTECODE="1")
        cmd = [sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-q", "-rfE", "--confcutdir", SUITE,
               "--rootdir", SUITE, "-o", "addopts=", *[os.path.join(SUITE, f) for f in files]]
        res = subprocess.run(cmd, cwd=tmp, env=env, capture_output=True, text=True, timeout=timeout)
    out = res.stdout + res.stderr
    failed = sorted(set(re.findall(r"^(?:FAILED|ERROR) \S*?(test_\w+\.py::[\w\[\].\-]+)", out, flags=re.M)))
    summary = [ln for ln in out.splitlines() if re.search(r"\d+ passed", ln)]
    return failed, (summary[-1] if summary else out[-3000:])


def _check(files, timeout):
    failed, summary = _run(files, timeout)
    print(f"reference suite {files}: {summary}")
    unexpected = [f for f in failed if f.split("[")[0] not in KNOWN]
    assert not unexpected, f"reference tests failing on the drop-in: {unexpected}\n{summary}"
    assert "passed" in summary


def test_reference_suite_host_modules():
    """mesh / quadrature: host code, no GPU needed."""
    _check(["test_mesh.py", "test_quadrature.py"], 900)


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_ok(), reason="needs a CUDA device")
def test_reference_suite_device_modules():
    """kernels / assembly / solver / postprocess / acceptance through the
    device path."""
    _check(["test_kernels.py", "test_assembly.py", "test_solver.py", "test_postprocess.py", "test_acceptance.py"],
           3000)
