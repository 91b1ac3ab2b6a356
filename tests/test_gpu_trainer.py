"""One optim::train iteration on the device (paper_2412_04459_b200.trainer):
render -> MSE + SSIM -> ray losses -> backward against the reference's own
composition of the same steps (optim.cpp:433-477), then the Adam updates
move the scene's device pools."""
import numpy as np
import pytest

from conftest import grad_close

pytestmark = pytest.mark.gpu


def test_train_iteration_gradients_match_reference(svr, ctx, ref):
    import torch
    from paper_2412_04459_b200.trainer import DeviceTrainer, TrainWeights
    arrays = svr.synth_random_scene(2024, 65536, 7, 3)
    scene = svr.Scene(ctx, arrays)
    rscene = ref.RefScene.generate(2024, 65536, 7, 3)
    cam = svr.ring_camera(1, 0, 96, 80)
    opts = svr.RenderOptions(K=2, supersample=1.5, training=True, background=(0.2, 0.1, 0.3))
    gt = np.random.default_rng(21).uniform(0, 1, (80, 96, 3))
    w = TrainWeights(lambda_T=0.05, lambda_dist=0.2, lambda_R=0.03)
    tr = DeviceTrainer(svr, ctx, scene, opts, w)
    gt_dev = torch.tensor(gt, dtype=torch.float32, device="cuda")
    log = tr.gradients(cam, gt_dev)
    losses_r, gd, gs, gp = ref.ref_train_iteration_grads(
        rscene, cam, opts, gt, w.lambda_ssim, w.lambda_T, w.lambda_dist, w.lambda_R,
        arrays.n_pool, arrays.n_voxels * arrays.sh_stride, arrays.n_voxels)
    ours = [log["l_mse"], log["l_ssim"], log["l_T"], log["l_dist"], log["l_R"]]
    np.testing.assert_allclose(ours, losses_r, rtol=1e-4, atol=1e-7)
    ctx.synchronize()
    for name, g, r in [("density", tr.g_density, gd), ("sh", tr.g_sh, gs),
                       ("priority", tr.g_priority, gp)]:
        nbad, worst = grad_close(g.cpu().numpy(), r)
        assert nbad == 0, f"{name}: {nbad} out of tolerance (worst excess {worst:.3e})"


def test_train_steps_update_pools_and_lower_loss(svr, ctx):
    import torch
    from paper_2412_04459_b200.trainer import DeviceTrainer
    arrays = svr.synth_random_scene(7, 20000, 7, 3)
    scene = svr.Scene(ctx, arrays)
    cam = svr.ring_camera(1, 0, 64, 64)
    opts = svr.RenderOptions(K=1, supersample=1.0)
    tr = DeviceTrainer(svr, ctx, scene, opts)
    gt = torch.full((64, 64, 3), 0.5, dtype=torch.float32, device="cuda")
    d0, s0 = tr.params()
    logs = [tr.step(cam, gt) for _ in range(30)]
    d1, s1 = tr.params()
    assert not np.array_equal(d0, d1) and not np.array_equal(s0, s1)
    assert logs[-1]["l_mse"] < 0.8 * logs[0]["l_mse"]
    assert float(tr.priority.sum()) > 0


def test_deferred_losses_match_immediate(svr, ctx):
    """Deferred mode (on_device = 2): the loss values read once with
    svr_frame_loss_values equal the immediately returned ones."""
    import torch
    from paper_2412_04459_b200.trainer import DeviceTrainer, TrainWeights
    arrays = svr.synth_random_scene(77, 20000, 7, 3)
    scene = svr.Scene(ctx, arrays)
    cam = svr.ring_camera(2, 1, 96, 80)
    gt = torch.tensor(np.random.default_rng(3).uniform(0, 1, (80, 96, 3)), dtype=torch.float32,
                      device="cuda")
    tr = DeviceTrainer(svr, ctx, scene, svr.RenderOptions(K=1, supersample=1.0),
                       TrainWeights(lambda_T=0.05, lambda_dist=0.2, lambda_R=0.03))
    now = tr.gradients(cam, gt)
    assert tr.gradients(cam, gt, defer=True) == {}
    later = tr.loss_values()
    for k, v in now.items():  # the block sums meet in double atomics: order-dependent last bits
        assert later[k] == pytest.approx(v, rel=1e-9, abs=1e-15), k
