"""The reference's OWN unit tests (spgemm_test.cpp, partition_test.cpp, scheduler_test.cpp) and its
release gate (acceptance.cpp), unmodified, compiled against the drop-in headers of include/aires/
(hot path on the B200, everything else the reference's) and linked to libaires_b200.so.  Built by
`make -C oracle dropin` where /root/reference exists (the binaries travel with the repo copy).
`real_test` (oracle/dropin_real_test.cpp) is ours: the real out-of-core run behind the same headers
(exact and streamed output, capped budgets, MaxMemory) against the in-core product, bit-exact."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("unit", ["spgemm_test", "partition_test", "scheduler_test", "gcn_test", "acceptance",
                                  "real_test"])
def test_reference_suite_on_b200(unit):
    exe = os.path.join(REF, f"dropin_{unit}")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time: make -C oracle dropin)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
