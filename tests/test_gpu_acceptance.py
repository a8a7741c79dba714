"""Drop-in check: the reference's own acceptance gate
(proj/tests/test_acceptance.cpp, unmodified) with its hot path served by
libkvt_b200.so through integration/kvtier_b200_shim.cpp (ELF interposition
in front of an -fPIC build of the reference library; oracle/Makefile target
test_acceptance_b200). Every replay, policy_insert, insert_joint,
rearrange and best_config in the gate runs on the GPU; the gate's golden
traces, greedy-vs-exact bound and capacity checks must all pass, exactly as
they do for the CPU build (oracle/_ref/test_acceptance)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GATE = os.path.join(ROOT, "oracle", "_ref", "test_acceptance_b200")

pytestmark = pytest.mark.gpu


def test_reference_acceptance_gate_on_b200():
    if not os.path.exists(GATE):
        pytest.skip("oracle/_ref/test_acceptance_b200 not built (needs /root/reference at build time)")
    env = dict(os.environ, KVT_SHIM_TRACE="1")
    r = subprocess.run([GATE], cwd=os.path.dirname(GATE), capture_output=True, text=True, timeout=900, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out
    assert out.count("[PASS]") == 9, out
    assert "[FAIL]" not in out, out
    # the shim really was in front of the reference library
    served = [l for l in out.splitlines() if l.startswith("kvt_b200 shim:")]
    assert served and int(served[-1].split()[2]) > 1000, out
