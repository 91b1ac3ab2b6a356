"""The CTA-cooperative composite (K7', raster.cu composite_coop_kernel) on the
parity cases of the forward and backward suites.

Frames choose between the warp-autonomous and the cooperative composite by
their mean entries per tile (SVR_COOP_MIN, read once per process), so on the
small scenes of the parity suites only the warp-autonomous kernel runs. Here
a child pytest re-runs those cases with SVR_COOP_MIN=0, which sends every
frame through the cooperative kernel: every compositing mode (plain render,
record pass, max-blend stats, staged training render), K = 1..3, supersampled
and non-multiple-of-16 images, opaque and constant-density voxels, deferred
frames, and the backward walks that consume its records — against the same
reference values and tolerances (raster.cpp:17-61, 238-281; 303-423).
"""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FORWARD = ("render_matches_reference or supersampled or small_scenes or record_stats or opaque "
           "or constant_density or empty_scene or async_downloads or deferred or outputs_block")


def _child(args):
    env = dict(os.environ, SVR_COOP_MIN="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-m", "gpu", "-q", "-p", "no:cacheprovider"] + args,
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout[-4000:] + r.stderr[-2000:]
    assert r.returncode == 0, out
    assert " passed" in r.stdout and " failed" not in r.stdout, out


def test_forward_parity_on_the_cooperative_composite():
    _child(["tests/test_gpu_forward.py", "-k", FORWARD])


def test_backward_parity_on_the_cooperative_composite():
    _child(["tests/test_gpu_backward.py", "tests/test_gpu_losses.py"])


def test_threshold_selects_the_cooperative_composite():
    """The frame reports the composite it ran (svr_frame_info.composite_path):
    cooperative under SVR_COOP_MIN=0, warp-autonomous on the same small frame
    at the default threshold."""
    code = ("import numpy as np, paper_2412_04459_b200 as svr\n"
            "ctx = svr.Context(0)\n"
            "a = svr.synth_random_scene(3, 1 << 14, 7, 2)\n"
            "sc = svr.Scene(ctx, a)\n"
            "f = svr.Frame(ctx)\n"
            "svr.render_into(f, sc, svr.ring_camera(4, 1, 200, 150), svr.RenderOptions(supersample=1.0))\n"
            "print('PATH', f.info().composite_path)\n")
    for env_val, want in (("0", 1), (None, 0)):
        env = dict(os.environ)
        env.pop("SVR_COOP_MIN", None)
        if env_val is not None:
            env["SVR_COOP_MIN"] = env_val
        r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        assert f"PATH {want}" in r.stdout, (env_val, r.stdout)
