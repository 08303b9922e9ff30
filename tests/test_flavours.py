"""The other two flavours of libsacd (paper_2003_03572_b200/build.py), each run in a
subprocess because the binding loads one library per process (SACD_LIB):
  * libsacd_debug.so (-DSACD_DEBUG): device-side asserts on every nonzero's a / b index, the
    row ids, work-item bounds and the partial / fix-up slots of the MTTKRP (compute-sanitizer
    is closed on the GPU pool, so this is the memory-safety check), on ragged tensors through
    every kernel family, with oracle parity;
  * libsacd_tuning.so (-DSACD_TUNING): the measured MTTKRP tuning variants kept out of the
    product library, each bitwise equal to the default kernel."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.mark.parametrize("flavour", ["debug", "tuning"])
def test_flavour(flavour):
    from paper_2003_03572_b200 import build
    lib = build.build(flavour=flavour)
    env = dict(os.environ, SACD_LIB=os.path.basename(lib))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_flavour_checks.py"), flavour], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=1500)
    print(r.stdout[-3000:])
    assert r.returncode == 0 and "FLAVOUR CHECKS PASSED" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
