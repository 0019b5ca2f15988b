"""Out-of-bounds checks of our own over every kernel of libmsrep (guard bands), and, opt-in,
compute-sanitizer.

test_guard_bands runs tests/sanitize_worker.py directly: every output buffer (y, SpMM Y, mirror
copies) sits inside a larger allocation whose leading and trailing 4096 elements hold a sentinel, and
the worker checks that no store landed there and that every result is bit-exact against the oracle.
The GPU pool this repo is tested on has compute-sanitizer CLOSED (runs under it left GPUs needing a
reset), so test_compute_sanitizer only runs with MSREP_SANITIZER=1 on a box where the tool is allowed.

compute-sanitizer over every kernel of libmsrep at small sizes: memcheck
(out-of-bounds / misaligned accesses, including the 1-D TMA bulk copies), racecheck (shared-memory
hazards between the warps of the pCSC band kernel and within the per-warp tile rings), synccheck
(barrier misuse: the named barriers of the pCSC consumers, __syncwarp masks, cluster barriers).
tests/sanitize_worker.py runs the cases and checks their results against the oracle.

racecheck does not model mbarrier phase completion (cp.async.bulk complete_tx + try_wait, and the
producer/consumer stage protocol built on it), so it reports the stage hand-offs of the TMA rings as
hazards.  Those -- and only those -- are accepted: every reported hazard must involve the 1-D TMA
copy (tma_1d) or be the pCSC producer's stage write (its `stage` lambda) against a consumer's
cb_load.  Anything else fails the test."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _mbarrier_protocol(block):
    if "tma_1d" in block:
        return True
    return "cb_load" in block and "csc_band_kernel" in block and "operator ()" in block


def test_guard_bands():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_worker.py")], capture_output=True,
                       text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "sanitize worker: OK" in out, out[-4000:]


@pytest.mark.skipif(os.environ.get("MSREP_SANITIZER") != "1",
                    reason="compute-sanitizer is closed on the GPU pool; opt in with MSREP_SANITIZER=1")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    cmd = [cs, f"--tool={tool}", "--print-limit=100000", sys.executable, os.path.join(ROOT, "tests", "sanitize_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=2400, cwd=ROOT)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log"), "w") as f:
        f.write(out)
    assert "sanitize worker: OK" in out, out[-4000:]
    if tool == "racecheck":
        blocks = re.split(r"=+ (?:Error|Warning): Race reported", out)[1:]
        bad = [b for b in blocks if not _mbarrier_protocol(b)]
        assert not bad, "racecheck hazards outside the mbarrier stage protocol:\n" + "\n".join(b[:1500] for b in bad[:5])
    else:
        assert r.returncode == 0, out[-6000:]
        assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
