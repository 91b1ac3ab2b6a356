"""Per-ray losses on the device: svr_ray_losses against
the unmodified reference ray_losses (losses.cpp:141-238) on identical
frames, then through render_backward as the reference training step uses
them (optim.cpp:439-471). Mirrors test_losses.cpp:130-238."""
import numpy as np
import pytest

from conftest import grad_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene1(svr, ctx, ref):
    arrays = svr.synth_random_scene(2024, 65536, 7, 3)
    return arrays, svr.Scene(ctx, arrays), ref.RefScene.generate(2024, 65536, 7, 3)


def sizes(a):
    return a.n_pool, a.n_voxels * a.sh_stride, a.n_voxels


def assert_grads(ours, theirs, label):
    nbad, worst = grad_close(ours, theirs)
    assert nbad == 0, f"{label}: {nbad} elements out of tolerance (worst excess {worst:.3e})"


@pytest.mark.parametrize("K,ss,w", [(1, 1.0, (0.3, 0.7, 0.2)), (2, 1.5, (0.1, 1.0, 0.5)),
                                    (3, 1.0, (0.0, 0.4, 0.0)), (1, 1.5, (0.5, 0.0, 0.0))])
def test_ray_losses_match_reference(svr, ctx, ref, scene1, K, ss, w):
    arrays, scene, rscene = scene1
    cam = svr.ring_camera(1, 0, 96, 80)
    opts = svr.RenderOptions(K=K, supersample=ss, training=True)
    gt = np.random.default_rng(5).uniform(0, 1, (80, 96, 3))
    rf = ref.RefFrame(rscene, cam, opts)
    vals_r, dtf_r, dw_r, dvc_r = rf.ray_losses(gt, *w)
    out = svr.render(scene, cam, opts)
    vals, dtf, dw, dvc = svr.ray_losses(out.frame, gt, *w)
    for name, a, b in zip(("l_T", "l_dist", "l_R"), vals, vals_r):
        assert abs(a - b) <= 1e-4 * abs(b) + 1e-9, f"{name}: {a} vs {b}"
    if w[0]:
        assert_grads(dtf, dtf_r, "d_tfin_ss")
    if w[1] or w[2]:
        assert_grads(dw, dw_r, "d_weight")
    if w[2]:
        # d_voxel_color = 2 w_R w (c - g) / rays: where c ~ g its error is the
        # absolute error of the fp32 voxel colour itself (forward tolerance
        # 1e-4); allow 1e-5 of colour error on top of the relative rule
        rays = (ss * 96) * (ss * 80)
        floor = 2.0 * w[2] / rays * 1e-5
        bad = np.abs(dvc - dvc_r) > 1e-3 * (np.maximum(np.abs(dvc), np.abs(dvc_r)) +
                                            1e-3 * np.abs(dvc_r).max()) + floor
        assert int(bad.sum()) == 0, f"d_voxel_color: {int(bad.sum())} elements out of tolerance"


def test_ray_losses_accumulate_into_given_buffers(svr, ctx, scene1):
    """Gradients add to what the buffers hold (UpstreamGrads semantics)."""
    arrays, scene, _ = scene1
    cam = svr.ring_camera(1, 0, 64, 64)
    out = svr.render(scene, cam, svr.RenderOptions(K=1, supersample=1.0, training=True))
    gt = np.random.default_rng(2).uniform(0, 1, (64, 64, 3))
    _, dtf, dw, dvc = svr.ray_losses(out.frame, gt, 0.2, 0.3, 0.4)
    _, dtf2, dw2, dvc2 = svr.ray_losses(out.frame, gt, 0.2, 0.3, 0.4, dtf.copy(), dw.copy(),
                                        dvc.reshape(-1).copy())
    np.testing.assert_allclose(dtf2, 2 * dtf, rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(dw2, 2 * dw, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(dvc2, 2 * dvc, rtol=1e-6, atol=1e-12)


def test_ray_losses_through_backward(svr, ctx, ref, scene1):
    """L1 + ray losses -> render_backward: the device step's gradients match
    the reference backward fed by the reference's own ray-loss upstreams."""
    arrays, scene, rscene = scene1
    cam = svr.ring_camera(1, 0, 96, 96)
    opts = svr.RenderOptions(K=2, supersample=1.0, training=True)
    gt = np.random.default_rng(9).uniform(0, 1, (96, 96, 3))
    w = (0.1, 0.5, 0.3)
    rf = ref.RefFrame(rscene, cam, opts)
    _, dtf_r, dw_r, dvc_r = rf.ray_losses(gt, *w)
    dcol = np.sign(rf.color - gt) / rf.color.size
    theirs = rf.backward(*sizes(arrays), d_color=dcol, d_tfin_ss=dtf_r, d_weight=dw_r,
                         d_voxel_color=dvc_r)
    out = svr.render(scene, cam, opts)
    _, dtf, dw, dvc = svr.ray_losses(out.frame, gt, *w)
    ours = svr.render_backward(scene, out.frame, d_color=dcol, d_tfin_ss=dtf, d_weight=dw,
                               d_voxel_color=dvc)
    for name, g, gr in [("density", ours.density, theirs[0]), ("sh", ours.sh, theirs[1]),
                        ("priority", ours.priority, theirs[2])]:
        assert_grads(g, gr, name)


def test_ray_losses_need_records(svr, ctx, scene1):
    arrays, scene, _ = scene1
    out = svr.render(scene, svr.ring_camera(1, 0, 32, 32), svr.RenderOptions(supersample=1.0))
    with pytest.raises(RuntimeError):
        svr.ray_losses(out.frame, np.zeros((32, 32, 3)), 0.1, 0.1, 0.1)


@pytest.mark.parametrize("w_mse,w_ssim", [(1.0, 0.02), (0.0, 1.0), (0.7, 0.0)])
def test_image_losses_match_reference(svr, ctx, ref, scene1, w_mse, w_ssim):
    """mse_loss + ssim_loss (losses.cpp:71-139) on the rendered colour."""
    arrays, scene, _ = scene1
    cam = svr.ring_camera(1, 0, 80, 64)
    out = svr.render(scene, cam, svr.RenderOptions(supersample=1.0))
    gt = np.random.default_rng(4).uniform(0, 1, (64, 80, 3))
    (mse_r, ssim_r), d_r = ref.ref_image_losses(out.color.astype(np.float64), gt, w_mse, w_ssim)
    (mse, ssim_l), d = svr.image_losses(out.frame, gt, w_mse, w_ssim)
    assert abs(mse - mse_r) <= 1e-6 * mse_r
    assert abs(ssim_l - ssim_r) <= 1e-5
    nbad, worst = grad_close(d, d_r)
    assert nbad == 0, f"d_color: {nbad} out of tolerance (worst excess {worst:.3e})"


def test_image_losses_reject_small_images(svr, ctx, scene1):
    arrays, scene, _ = scene1
    out = svr.render(scene, svr.ring_camera(1, 0, 10, 40), svr.RenderOptions(supersample=1.0))
    with pytest.raises(ValueError):
        svr.image_losses(out.frame, np.zeros((40, 10, 3)), 1.0, 1.0)
