"""Run the reference's OWN test suite (pkg/tests, installed next to the
reference under baseline/_ref by baseline/install_ref.sh) with the GPU path
plugged into the reference (paper_2508_02613_b200.plugin.plug_into_reference):
every operator / preconditioner / solver binding site of ``jfft`` is rebound
to libjfftb200 before the tests import the package, so the reference's tests
exercise the CUDA library through the reference's own API.

    python tests/run_reference_suite.py [pytest args...]

Writes gpurun_out/reference_suite.json ({test id: outcome}) and exits with
pytest's status.  Used by tests/test_gpu_reference_suite.py.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF = os.path.join(REPO, "baseline", "_ref")


class _Plugin:
    """pytest plugin: plug the GPU path in before collection, record outcomes."""

    def __init__(self):
        self.outcomes = {}

    def pytest_configure(self, config):
        import jfft  # noqa: F401  (the installed reference)
        from paper_2508_02613_b200.plugin import plug_into_reference
        plug_into_reference("jfft")

    def pytest_runtest_logreport(self, report):
        if report.when == "call" or report.outcome != "passed":
            self.outcomes[report.nodeid] = report.outcome


def main(argv) -> int:
    import pytest
    if not os.path.isdir(os.path.join(REF, "tests")):
        print(f"{REF}/tests missing: run baseline/install_ref.sh", file=sys.stderr)
        return 2
    sys.path[:0] = [REF, os.path.join(REF, "tests"), REPO]
    plug = _Plugin()
    rc = pytest.main([os.path.join(REF, "tests"), "-q", "-p", "no:cacheprovider",
                      "--rootdir", REF, *argv], plugins=[plug])
    out = os.path.join(REPO, "gpurun_out", "reference_suite.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        json.dump(plug.outcomes, fh, indent=1, sort_keys=True)
    return int(rc)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
