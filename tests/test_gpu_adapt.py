"""Scene adaptation on the device against the
unmodified reference prune / subdivide_voxels (optim.cpp:207-298) with
rebuild_corner_indexing (scene.cpp:8-26): voxels, corner indexing (pool
order), densities (incl. the fresh subdivision averages), SH rows and the
AdaptRemap, bit for bit. Mirrors test_optim.cpp's adaptation cases."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scenes(svr, ctx, ref):
    arrays = svr.synth_random_scene(2024, 30000, 7, 3)
    return arrays, svr.Scene(ctx, arrays), ref.RefScene.generate(2024, 30000, 7, 3)


def assert_same(ours, theirs, vs, ps, vs_r, ps_r):
    a, r = ours.arrays, theirs.arrays()
    assert a.n_voxels == r.n_voxels and a.n_pool == r.n_pool
    for name in ("codes", "levels", "corner_index", "density", "sh"):
        assert np.array_equal(getattr(a, name), getattr(r, name)), name
    assert np.array_equal(vs, vs_r) and np.array_equal(ps, ps_r)


@pytest.mark.parametrize("thr", [0.0, 0.3, 0.9, 2.0])
def test_prune_matches_reference(svr, ctx, ref, scenes, thr):
    arrays, scene, rscene = scenes
    stats = np.random.default_rng(7).uniform(0, 1, arrays.n_voxels).astype(np.float32)
    ours = scene.prune(stats, thr)
    theirs, vs_r, ps_r = ref.ref_adapt(rscene, prune_stats=stats.astype(np.float64), threshold=thr)
    assert_same(ours, theirs, *ours.remap(), vs_r, ps_r)


@pytest.mark.parametrize("frac,seed", [(0.0, 1), (0.01, 2), (0.05, 3), (0.3, 4)])
def test_subdivide_matches_reference(svr, ctx, ref, scenes, frac, seed):
    arrays, scene, rscene = scenes
    rng = np.random.default_rng(seed)
    sel = rng.choice(arrays.n_voxels, int(frac * arrays.n_voxels), replace=False).astype(np.uint32)
    sel = np.concatenate([sel, sel[:5]])  # duplicates are ignored
    ours = scene.subdivide(sel)
    theirs, vs_r, ps_r = ref.ref_adapt(rscene, selected=sel)
    assert_same(ours, theirs, *ours.remap(), vs_r, ps_r)


def test_adapted_scene_renders_like_reference(svr, ctx, ref, scenes):
    arrays, scene, rscene = scenes
    rng = np.random.default_rng(11)
    sel = rng.choice(arrays.n_voxels, 800, replace=False).astype(np.uint32)
    ours = scene.subdivide(sel).prune(rng.uniform(0, 1, arrays.n_voxels + 7 * 800), 0.05)
    cam = svr.ring_camera(1, 0, 64, 64)
    o = svr.RenderOptions(supersample=1.0)
    a = ours.arrays
    r = ref.ref_render(ref.RefScene.from_arrays(a), cam, o)
    out = svr.render(ours, cam, o)
    assert float(np.max(np.abs(out.color - r["color"]))) <= 1e-4


def test_adaptation_errors(svr, ctx, scenes):
    arrays, scene, _ = scenes
    with pytest.raises(ValueError):
        scene.prune(np.zeros(3, np.float32), 0.1)
    with pytest.raises(ValueError):
        scene.subdivide([arrays.n_voxels])
