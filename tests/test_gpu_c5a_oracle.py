"""c5a one-step parity vs the C++ oracle on element 0.  Several minutes of fp64 CPU work:
runs only with LD_SLOW_TESTS=1 (evidence: profiles/r02_c5a_oracle_check.json)."""
import os

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(3600)
@pytest.mark.skipif(os.environ.get("LD_SLOW_TESTS") != "1", reason="slow: set LD_SLOW_TESTS=1")
def test_c5a_step_element0_vs_cpp_oracle():
    from tests.tools.c5a_oracle_check import main
    out = main(1)
    assert out["rel_l2"] < 2e-3
