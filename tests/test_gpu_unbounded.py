"""Config-4/5 scene (init_unbounded, 7,824,544 voxels over levels 2-16) on the
GPU: cameras inside the scene, so near-plane straddlers get the whole image
(raster.cpp:95-101) and tiles carry several sign patterns. Bit-exact entry
list, sort order and ranges against the unmodified reference at a resolution
the CPU finishes in seconds; images within 1e-4. The full 1024^2 views are
bench workloads (E ~ 90M per view): there the sorted keys are checked for
order and the ranges for consistency on the device."""
import numpy as np
import pytest

from conftest import max_abs, sentinel_aware_depth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def cfg4(svr, ctx, ref):
    cams = [svr.ring_camera(8, i, 1024, 1024) for i in range(8)]
    arrays = svr.synth_unbounded_scene(cams, 7, 5, 2.8, seed=7)
    assert (arrays.n_voxels, arrays.n_pool) == (7824544, 16227695)
    return arrays, svr.Scene(ctx, arrays), ref.RefScene.from_arrays(arrays)


@pytest.mark.parametrize("view", [0, 77])
def test_cfg4_entries_sort_ranges_bit_exact(svr, ctx, ref, cfg4, view):
    arrays, scene, rscene = cfg4
    cam = svr.ring_camera(256, view, 96, 96, 1.0)
    f = svr.Frame(ctx)
    svr.render_into(f, scene, cam, svr.RenderOptions(supersample=1.0))
    k_ref, v_ref = ref.ref_entries(rscene, cam, sorted_=False)
    assert f.info().n_entries == k_ref.size > 0
    assert np.array_equal(f.download("ENTRIES_KEYS", np.uint64), k_ref)
    assert np.array_equal(f.download("ENTRIES_VALUES", np.uint32), v_ref)
    ks_ref, vs_ref = ref.ref_entries(rscene, cam, sorted_=True)
    assert np.array_equal(f.download("SORT_KEYS", np.uint64), ks_ref)
    assert np.array_equal(f.download("SORT_VALUES", np.uint32), vs_ref)
    ranges = f.download("TILE_RANGES", np.uint32, (-1, 2))
    tiles = (ks_ref >> np.uint64(48)).astype(np.int64)
    lo = np.searchsorted(tiles, np.arange(ranges.shape[0]), "left")
    hi = np.searchsorted(tiles, np.arange(ranges.shape[0]), "right")
    ne = hi > lo
    assert np.array_equal(ranges[ne, 0], lo[ne]) and np.array_equal(ranges[ne, 1], hi[ne])


def test_cfg4_images_match_reference(svr, ctx, ref, cfg4):
    arrays, scene, rscene = cfg4
    cam = svr.ring_camera(256, 5, 64, 64, 1.0)
    opts = svr.RenderOptions(supersample=1.0)
    out = svr.render(scene, cam, opts)
    r = ref.ref_render(rscene, cam, opts)
    assert max_abs(out.color, r["color"]) <= 1e-4
    assert max_abs(out.transmittance, r["transmittance"]) <= 1e-4
    assert max_abs(out.normal, r["normal"]) <= 1e-4
    assert sentinel_aware_depth(out.depth, r["depth"]) <= 1e-4


def test_cfg4_full_view_order_properties(svr, ctx, cfg4):
    """1024^2 view (E ~ 9e7): keys ascending, values a permutation-consistent
    decode, ranges tile the list without gaps."""
    arrays, scene, _ = cfg4
    f = svr.Frame(ctx)
    svr.render_into(f, scene, svr.ring_camera(256, 0, 1024, 1024, 1.0),
                    svr.RenderOptions(supersample=1.0))
    E = f.info().n_entries
    assert E > 40_000_000
    k = f.download("SORT_KEYS", np.uint64)
    assert k.size == E and bool(np.all(k[1:] >= k[:-1]))
    v = f.download("SORT_VALUES", np.uint32)
    assert int((v & ((1 << 29) - 1)).max()) < arrays.n_voxels
    ranges = f.download("TILE_RANGES", np.uint32, (-1, 2)).astype(np.int64)
    ne = ranges[:, 1] > ranges[:, 0]
    r = ranges[ne][np.argsort(ranges[ne, 0])]
    assert r[0, 0] == 0 and r[-1, 1] == E and np.array_equal(r[1:, 0], r[:-1, 1])
    tiles = (k[r[:, 0]] >> np.uint64(48)).astype(np.int64)
    assert np.array_equal(np.flatnonzero(ne)[np.argsort(ranges[ne, 0])], tiles)


@pytest.mark.parametrize("huge_min", ["2", "9", "40"])
def test_huge_pair_merge_matches_full_sort(svr, ref, monkeypatch, huge_min):
    """The huge-pair merge (production frames: pairs covering >= SVR_HUGE_MIN
    tiles are merged into the tile lists by rank instead of duplicated and
    sorted) yields exactly the reference's sorted values and tile ranges, and
    images identical to the unmerged path, on a camera inside a small scene
    (thresholds lowered so most pairs take the merge)."""
    import numpy as np
    arrays = svr.synth_random_scene(77, 512 + 7 * 300, 8, 2)
    rscene = ref.RefScene.from_arrays(arrays)
    cam = svr.Camera(160, 112, 60.0, 60.0, 79.3, 55.7, np.eye(3), np.array([0.01, -0.02, -0.03]))
    opts = svr.RenderOptions(supersample=1.0)
    ks, vs = ref.ref_entries(rscene, cam, sorted_=True)
    monkeypatch.setenv("SVR_HUGE_MIN", "0")
    plain = svr.Context(0)
    base = svr.render(svr.Scene(plain, arrays), cam, opts)
    monkeypatch.setenv("SVR_HUGE_MIN", huge_min)
    ctx = svr.Context(0)
    scene = svr.Scene(ctx, arrays)
    f = svr.Frame(ctx)
    for _ in range(2):  # the first frame counts the huge pairs, the second merges them
        out = svr.render(scene, cam, opts, frame=f)
    assert f.info().n_entries == ks.size
    assert np.array_equal(f.download("SORT_VALUES", np.uint32), vs)
    ranges = f.download("TILE_RANGES", np.uint32, (-1, 2))
    tiles = (ks >> np.uint64(48)).astype(np.int64)
    t = np.arange(ranges.shape[0])
    lo, hi = np.searchsorted(tiles, t, "left"), np.searchsorted(tiles, t, "right")
    ne = hi > lo
    assert np.array_equal(ranges[ne, 0], lo[ne]) and np.array_equal(ranges[ne, 1], hi[ne])
    for name in ("color", "depth", "median_depth", "normal", "transmittance"):
        assert np.array_equal(getattr(out, name), getattr(base, name)), name
