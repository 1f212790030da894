"""The reference's OWN test suite, run against the GPU path (SURVEY §4,
implication 2): ``integration/conegrad_plugin.py`` installs the binding
``integration/conegrad_cuda.py`` into the unmodified reference installed in
baseline/_ref (baseline/install_ref.sh), so every ``conegrad.jvp`` / ``vjp``
/ ``check_solution`` call of those modules runs on the B200 through the C
ABI.  Suites (reference files):

* tests/test_solution_map.py -- encode/decode, dense-KKT oracle
  (:267-303), exact dP symmetry and duality (:396-431), pre-check errors;
* tests/test_acceptance.py -- criteria 1-8 (4: adjoints and duality, 5:
  oracle triangulation, 6: vjp mask, 8: CLI goldens);
* tests/test_golden.py -- the committed jvp/vjp goldens through the CLI,
  relaxed to 1e-6 and +-3 LSMR iterations as SURVEY §8(c) prescribes.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITES = ["test_solution_map.py", "test_acceptance.py", "test_golden.py"]


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")),
                    reason="reference not installed (baseline/install_ref.sh)")
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_gpu(suite):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "integration"), ROOT,
                                         env.get("PYTHONPATH", "")])
    env.setdefault("OPENBLAS_NUM_THREADS", "1")
    log_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(log_dir, exist_ok=True)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "conegrad_plugin", "-p", "no:cacheprovider",
                        "--rootdir", os.path.join(REF, "tests"), os.path.join(REF, "tests", suite)],
                       cwd=os.path.join(REF, "tests"), env=env, capture_output=True, text=True, timeout=1800)
    with open(os.path.join(log_dir, f"refsuite_{suite.replace('.py', '')}.log"), "w") as f:
        f.write(r.stdout + "\n" + r.stderr)
    tail = "\n".join(r.stdout.strip().splitlines()[-25:])
    assert r.returncode == 0, f"reference suite {suite} on the GPU path failed:\n{tail}\n{r.stderr[-2000:]}"
    assert "libqcpgrad" in r.stdout or "passed" in r.stdout
