"""Drop-in boundary, end to end: the reference's own
integrators (proj/src/integrators.cpp, unmodified, in oracle/_ref) drive the
B200 library through the C++ shim a maintainer adds (integration/
eqs_gpu_shim.hpp), next to the reference's FemSystem on the
same problem built by the reference. integration/_build/dropin_main is built
where the reference sources exist (__graft_entry__.build) and travels to the
GPU box with the snapshot."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "dropin_main")


@pytest.mark.skipif(not os.path.exists(BIN), reason="integration/_build/dropin_main not built (no reference sources)")
def test_reference_integrators_through_the_shim():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    line = out.stdout.strip().splitlines()[-1]
    r = json.loads(line)
    assert out.returncode == 0 and r["pass"], line
    assert r["rel_eval_rhs"] <= 1e-9
    assert r["rel_10_fixed_rkc_steps"] <= 1e-9
    assert r["same_accept_and_stages"] == 1
    assert r["sdirk_converged"] == [1, 1] and r["rel_2_fixed_sdirk_steps"] <= 1e-7
    assert r["sdirk_newton_solves_gpu"] == r["sdirk_newton_solves_reference"]
