"""GPU parity of the gradient path against the unmodified reference.

Per-element rule of SURVEY §8(c): |g-g_ref| <= 1e-3*(max(|g|,|g_ref|) + s),
s = 1e-3*max|g_ref|. Identical upstream gradients are fed to both sides
(the reference's L1 gradient), then the fused GPU train step is checked end
to end. Mirrors test_raster.cpp:413-557 and test_losses.cpp.
"""
import numpy as np
import pytest

from conftest import untie_gt, grad_close, look_at_origin, max_abs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene1(svr, ctx, ref):
    arrays = svr.synth_random_scene(2024, 65536, 7, 3)
    return arrays, svr.Scene(ctx, arrays), ref.RefScene.generate(2024, 65536, 7, 3)


def check_grads(ours, theirs, label):
    for name, g, gr in [("density", ours.density, theirs[0]), ("sh", ours.sh, theirs[1]),
                        ("priority", ours.priority, theirs[2])]:
        nbad, worst = grad_close(g, gr)
        assert nbad == 0, f"{label}/{name}: {nbad} elements out of tolerance (worst excess {worst:.3e})"


def sizes(a):
    return a.n_pool, a.n_voxels * a.sh_stride, a.n_voxels


@pytest.mark.parametrize("K,ss", [(1, 1.0), (2, 1.0), (3, 1.0), (1, 1.5)])
def test_backward_identical_upstream(svr, ctx, ref, scene1, K, ss):
    arrays, scene, rscene = scene1
    cam = svr.ring_camera(1, 0, 160, 160)
    opts = svr.RenderOptions(K=K, supersample=ss, training=True, background=(0.15, 0.25, 0.1))
    rng = np.random.default_rng(17)
    gt = rng.uniform(0, 1, (cam.height, cam.width, 3))
    loss_ref, dcol, gd, gs, gp = ref.ref_train_step_l1(rscene, cam, opts, gt, *sizes(arrays))
    out = svr.render(scene, cam, opts)
    g = svr.render_backward(scene, out.frame, d_color=dcol)
    check_grads(g, (gd, gs, gp), f"K={K} ss={ss}")


@pytest.mark.parametrize("K", [1, 2])
def test_axis_aligned_rays_on_voxel_faces(svr, ctx, ref, scene1, K):
    """Camera on voxel faces with rays whose direction has exact zero
    components (row py = cy - 0.5, column px = cx - 0.5): ray_aabb's IEEE
    semantics (field.hpp:58-69) for the 0/0 slabs, forward and backward."""
    arrays, scene, rscene = scene1
    cam = svr.Camera(96, 80, 70.0, 70.0, 48.5, 40.5, np.eye(3), np.array([0.0, 0.0, -0.25]))
    opts = svr.RenderOptions(K=K, supersample=1.0, training=True)
    out = svr.render(scene, cam, opts)
    r = ref.ref_render(rscene, cam, opts)
    assert max_abs(out.color, r["color"]) <= 1e-4
    assert max_abs(out.transmittance, r["transmittance"]) <= 1e-4
    gt = np.random.default_rng(23).uniform(0, 1, (cam.height, cam.width, 3))
    loss_ref, dcol, gd, gs, gp = ref.ref_train_step_l1(rscene, cam, opts, gt, *sizes(arrays))
    g = svr.render_backward(scene, out.frame, d_color=dcol)
    check_grads(g, (gd, gs, gp), f"axis-aligned K={K}")


def test_backward_depth_normal_tfin_channels(svr, ctx, ref, scene1):
    arrays, scene, rscene = scene1
    cam = svr.ring_camera(2, 1, 96, 96)
    opts = svr.RenderOptions(K=3, supersample=1.0, training=True)
    rng = np.random.default_rng(19)
    rf = ref.RefFrame(rscene, cam, opts)
    wD = np.where(rf.depth < 1e20, rng.uniform(-1, 1, rf.depth.shape), 0.0)
    wN = rng.uniform(-1, 1, rf.normal.shape)
    wT = rng.uniform(-1, 1, rf.sw * rf.sh)
    theirs = rf.backward(*sizes(arrays), d_depth=wD, d_normal=wN, d_tfin_ss=wT)
    out = svr.render(scene, cam, opts)
    ours = svr.render_backward(scene, out.frame, d_depth=wD, d_normal=wN, d_tfin_ss=wT)
    check_grads(ours, theirs, "depth/normal/tfin")


def test_backward_per_contribution_upstreams(svr, ctx, ref, scene1):
    arrays, scene, rscene = scene1
    cam = svr.ring_camera(1, 0, 64, 64)
    opts = svr.RenderOptions(K=2, supersample=1.0, training=True)
    rf = ref.RefFrame(rscene, cam, opts)
    out = svr.render(scene, cam, opts)
    inf = out.frame.info()
    assert inf.n_contribs == rf.n_contribs
    rng = np.random.default_rng(3)
    dw = rng.uniform(-1, 1, rf.n_contribs)
    dvc = rng.uniform(-1, 1, (rf.n_contribs, 3))
    theirs = rf.backward(*sizes(arrays), d_weight=dw, d_voxel_color=dvc)
    ours = svr.render_backward(scene, out.frame, d_weight=dw, d_voxel_color=dvc)
    check_grads(ours, theirs, "d_weight/d_voxel_color")


def test_forward_records_match_reference(svr, ctx, ref, scene1):
    arrays, scene, rscene = scene1
    cam = svr.ring_camera(1, 0, 96, 80)
    opts = svr.RenderOptions(K=1, supersample=1.5, training=True)
    rf = ref.RefFrame(rscene, cam, opts)
    pre_r, cp_r, ca_r, cb_r, pb_r, pc_r, _ = rf.records()
    out = svr.render(scene, cam, opts)
    pre, cp, ca, cb, pb, pc = out.frame.records()
    assert np.array_equal(pre, pre_r)
    assert np.array_equal(pc, pc_r) and np.array_equal(pb, pb_r)
    assert np.array_equal(cp, cp_r)
    assert max_abs(ca, ca_r) < 1e-5 and max_abs(cb, cb_r) < 1e-5


def test_train_step_end_to_end(svr, ctx, ref, scene1):
    """cfg3 pattern at reduced size: forward -> L1 -> backward on the GPU,
    against the reference's own train step on the same ground truth (pixels
    within 1e-3 of the reference colour are moved off the L1 kink first, so
    the sign of C - gt is the same on both sides)."""
    import torch
    arrays, scene, rscene = scene1
    cam = svr.ring_camera(1, 0, 128, 128)
    opts = svr.RenderOptions(K=1, supersample=1.0, training=True)
    gt = np.random.default_rng(17).uniform(0, 1, (128, 128, 3))
    gt = untie_gt(gt, svr.render(scene, cam, opts).color)  # |C - C_ref| <= 1e-4
    loss_ref, dcol_ref, gd, gs, gp = ref.ref_train_step_l1(rscene, cam, opts, gt, *sizes(arrays))
    dev = torch.device("cuda", 0)
    gt_t = torch.tensor(gt, dtype=torch.float32, device=dev)
    gd_t = torch.zeros(arrays.n_pool, device=dev)
    gs_t = torch.zeros(arrays.n_voxels * arrays.sh_stride, device=dev)
    gp_t = torch.zeros(arrays.n_voxels, device=dev)
    loss_t = torch.zeros(1, device=dev)
    torch.cuda.synchronize()
    import ctypes as C
    g = svr.svr_gradients()
    g.density, g.sh, g.priority, g.on_device = gd_t.data_ptr(), gs_t.data_ptr(), gp_t.data_ptr(), 1
    f = svr.Frame(ctx)
    c, o = cam.to_c(), opts.to_c()
    svr._check(svr.load_library().svr_train_step_l1(ctx.h, scene.h, C.byref(c), C.byref(o),
                                                     gt_t.data_ptr(), f.h, C.byref(g), 0,
                                                     loss_t.data_ptr()))
    ctx.synchronize()
    assert abs(loss_t.item() - loss_ref) < 1e-5
    color = f.download("COLOR", np.float32, (128, 128, 3))
    assert np.array_equal(np.sign(color - gt.astype(np.float32)), np.sign(dcol_ref))
    for name, ours, theirs in [("density", gd_t, gd), ("sh", gs_t, gs), ("priority", gp_t, gp)]:
        nbad, worst = grad_close(ours.cpu().numpy(), theirs)
        assert nbad == 0, f"{name}: {nbad} out of tolerance (worst excess {worst:.3e})"


def test_zero_upstream_and_mismatch(svr, ctx, scene1):
    """test_raster.cpp:413-442."""
    arrays, scene, _ = scene1
    cam = look_at_origin(svr, 24, 24, 1.7, 0.5)
    out = svr.render(scene, cam, svr.RenderOptions(supersample=1.0, training=True))
    g = svr.render_backward(scene, out.frame)
    assert not g.density.any() and not g.sh.any() and not g.priority.any()
    n = out.frame.info().n_contribs
    assert n > 0
    with pytest.raises(svr.RuntimeErrorSvr):
        svr.render_backward(scene, out.frame, d_weight=np.zeros(n + 1))
    out2 = svr.render(scene, cam, svr.RenderOptions(supersample=1.0, training=False))
    with pytest.raises(svr.RuntimeErrorSvr):
        svr.render_backward(scene, out2.frame, d_color=np.zeros((24, 24, 3)))


def test_opaque_backward(svr, ctx, ref):
    """Opaque voxels (density 800, alpha == 1): the division-free recursion
    (raster.cpp:374-407) must still produce the reference gradients."""
    codes = np.array([0, 4 << 45, (2 << 42) | (0 << 45)], np.uint64)
    rs = ref.RefScene.from_paths(np.array([0, 4 << 45], np.uint64), np.array([1, 1], np.uint8), 0.0, 1)
    a = rs.arrays()
    rng = np.random.default_rng(1)
    a.density[:] = rng.uniform(-0.3, 1.7, a.n_pool).astype(np.float32)
    a.density[0] = 800.0
    a.sh[:, :3] = (0.3 + 0.5 * rng.uniform(0, 1, (a.n_voxels, 3))) / 0.28209479177387814
    a.sh[:, 3:] = 0.05 * (rng.uniform(0, 1, (a.n_voxels, a.sh_stride - 3)) - 0.5)
    rs.set_params(a.density, a.sh)
    scene = svr.Scene(ctx, a)
    cam = look_at_origin(svr, 24, 24, 1.9, 0.6, 0.2)
    opts = svr.RenderOptions(K=2, supersample=1.0, training=True, background=(0.15, 0.25, 0.1))
    gt = rng.uniform(0, 1, (24, 24, 3))
    _, dcol, gd, gs, gp = ref.ref_train_step_l1(rs, cam, opts, gt, *sizes(a))
    out = svr.render(scene, cam, opts)
    check_grads(svr.render_backward(scene, out.frame, d_color=dcol), (gd, gs, gp), "opaque")
