"""The large-nx slice-phase paths on small golden cases.

Slices whose vectors do not fit in shared memory (cfg4's nx = 8192) keep them
in global memory and run the slice phase on every CTA of the cluster (element
loops, flip lifts, list counters through DSMEM, cluster scans), with the field
scan in an on-chip buffer or staged through a TMA ring.  The golden cases are
small, so they would take the on-chip paths; the library's test hook
PK_FORCE_GLOBAL_SLICE (read once per process) forces the global ones, and the
same bitwise tests run again in a child process."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# hybrid goldens with flips (lift and zero re-initialisation), eps(x), stale
# neighbours, the guard, parareal runs and 3V hybrid cases
SELECT = [
    "tests/test_gpu_parity.py::test_hybrid_golden",
    "tests/test_gpu_parity.py::test_eps_profile_hybrid_vs_oracle",
    "tests/test_gpu_parity.py::test_stale_neighbour_semantics",
    "tests/test_gpu_parity.py::test_all_kinetic_hybrid_equals_kinetic",
    "tests/test_gpu_parity.py::test_invalid_reinit_raises_on_flip",
    "tests/test_gpu_parity.py::test_parareal_small_golden",
    "tests/test_gpu_parity.py::test_batched_fine_matches_serial_windows",
    "tests/test_v3.py::test_v3_kinetic_lift_hybrid_golden",
]


@pytest.mark.parametrize("mode", ["1", "2"], ids=["scan-buffer", "staged-scan"])
def test_golden_cases_through_global_slice_paths(mode):
    env = dict(os.environ, PK_FORCE_GLOBAL_SLICE=mode)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "-m", "gpu", *SELECT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert " passed" in r.stdout
