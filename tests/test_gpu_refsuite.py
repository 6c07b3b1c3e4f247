"""The reference's OWN test-suite, unmodified, against this package.

`__graft_entry__.build()` stages pkg/tests of the reference into the git-ignored
baseline/_ref/_tests (next to the pip-installed reference that bench.py times); it travels to the
GPU box with the snapshot. tests/refsuite/orcasim is a package of re-exports that binds the name
`orcasim` (and orcasim.engine / .lp / .orca / .grid / .scenario / .crossings / .cli / .bench /
._kernels) to paper_2008_11578_b200, so every `from orcasim... import ...` of those tests lands
in the GPU implementation: 102 tests of desired velocities, single steps, mirror symmetries,
run-level properties, determinism across worker counts, the composed public operations against
`step`, grids and neighbour queries, the LP against enumeration / grid oracles, VO exits against
boundary sampling, scenario parsing, spawn sampling, trajectory files and the CLI.

Nothing here reads /root/reference; where the suite was not staged the test is skipped."""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "_tests")
SHIM = os.path.join(ROOT, "tests", "refsuite")


def run_suite(extra=()):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([SHIM, ROOT] + ([env["PYTHONPATH"]] if env.get("PYTHONPATH") else []))
    return subprocess.run([sys.executable, "-m", "pytest", SUITE, "-q", "-p", "no:cacheprovider", "-rf", *extra],
                          capture_output=True, text=True, env=env, cwd=ROOT, timeout=3000)


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="the reference's test-suite is not staged (baseline/_ref/_tests)")
def test_reference_suite_passes_against_this_package():
    out = run_suite()
    tail = "\n".join(out.stdout.strip().splitlines()[-40:])
    m = re.search(r"(\d+) passed", out.stdout)
    assert out.returncode == 0, tail
    assert m and int(m.group(1)) >= 102, tail
