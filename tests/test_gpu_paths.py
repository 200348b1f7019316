"""Every alternative device path, forced on the small golden cases.

The runtime picks kernels by size (cluster vs. cooperative CPQR, shared vs.
global panel QR, one-shot vs. chunked front targets, ring vs. dedicated
upload buffers); the full-size configs exercise only some of them.  Each
switch below is read once per process, so each case re-runs the golden
parity tests of test_gpu_factor.py in a subprocess with the switch set."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SWITCHES = {
    "chunked_targets": {"SPQ_CHUNK_BYTES": "65536"},
    "global_panel": {"SPQ_PANEL_GLOBAL": "1"},
    "cooperative_cpqr": {"SPQ_CPQR_COOP": "1"},
    "cooperative_cpqr_global_maps": {"SPQ_CPQR_COOP": "1", "SPQ_CPQR_GMAPS": "1"},
    "no_cluster_cpqr": {"SPQ_CPQR_CLMAX": "0"},
    "legacy_cpqr_kernels": {"SPQ_CPQR_NOWS": "1"},
    "legacy_cpqr_no_cta": {"SPQ_CPQR_NOWS": "1", "SPQ_CPQR_CLUSTER": "1"},
    "small_upload_ring": {"SPQ_RING_SMALL": "1"},
    "gemm_v1": {"SPQ_GEMM": "1"},
    "exact_row_flags": {"SPQ_NO_SPEC": "1"},
    "sparsify_prefix_waves": {"SPQ_SPARSIFY_PREFIX": "1"},
    "legacy_panel_smem": {"SPQ_PANEL_LEGACY": "1"},
    "register_panel_512_rows": {"SPQ_PANEL_ROWS": "512"},
    "speculation_failure_retry": {"SPQ_SPEC_TEST_FAIL": "1"},
}


@pytest.mark.parametrize("name", sorted(SWITCHES))
def test_forced_path_matches_golden(name):
    env = dict(os.environ, **SWITCHES[name])
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_factor.py"),
           "-k", "C1_n24 or C3_n48 or C4_n12 or chain"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, f"{name}: {SWITCHES[name]}\n{r.stdout[-3000:]}\n{r.stderr[-2000:]}"
