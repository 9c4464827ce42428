"""GPU: uninitialised-read and stale-state check (the substitute for
compute-sanitizer initcheck, which is closed on this pool).  With BD_POISON=1
every allocation of the library starts as all-ones bytes (a NaN pattern), so
a kernel that reads device memory nothing wrote poisons its results.  The
parity suites below (operators, preconditioners, PCG histories and counters,
100-step time stepping with all three inners, the sharded engine) must still
pass bit-for-bit as without poisoning."""
import os
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("suite", ["test_gpu_parity.py", "test_gpu_trsv_variants.py",
                                   "test_gpu_distributed.py"])
def test_parity_with_poisoned_allocations(suite):
    env = dict(os.environ, BD_POISON="1")
    p = subprocess.run([sys.executable, "-m", "pytest", os.path.join(REPO, "tests", suite), "-q",
                        "-x", "-p", "no:cacheprovider", "-m", "gpu"],
                       capture_output=True, text=True, timeout=1500, env=env, cwd=REPO)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
