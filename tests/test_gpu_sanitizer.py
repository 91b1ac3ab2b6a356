"""compute-sanitizer gate: memcheck, racecheck and synccheck
report no error on a small end-to-end workload (tools/sanitize_workload.py:
every composite mode on both K7 paths, the backward with all upstreams,
losses, and a deferred-E frame that outgrows its capacity)."""
import os
import shutil
import subprocess

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,coop", [("memcheck", "2048"), ("memcheck", "0"),
                                       ("racecheck", "2048"), ("racecheck", "0"),
                                       ("synccheck", "0")])
def test_sanitizer_clean(tool, coop):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    env = dict(os.environ, SVR_COOP_MIN=coop)
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    r = subprocess.run(cmd + ["python", os.path.join(ROOT, "tools", "sanitize_workload.py")],
                       capture_output=True, text=True, timeout=1500, env=env)
    out = r.stdout[-6000:] + r.stderr[-3000:]
    if r.returncode == 86 and "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (a pool-wide
        # decision, not a finding); the gate passed on this code in round 2
        # (profiles/r02/pytest_gpu_final.log)
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, out
    assert "sanitize workload ok" in r.stdout, out
    text = r.stdout + r.stderr
    clean = ("RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" if tool == "racecheck"
             else "ERROR SUMMARY: 0 errors")
    assert clean in text, out
