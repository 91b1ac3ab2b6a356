"""SVRX checkpoints <-> device scenes, mirroring
test_io.cpp:167-219: byte identity with the reference's own save_checkpoint
(io.cpp:250-279, compiled unmodified into oracle/_ref), files crossing both
ways between the reference's load_checkpoint and ours, lossless round trip
with bit-identical renders, the empty scene, rejection of corrupted /
truncated / absent files with the reference's verdicts, and a checkpoint of
parameters a device training step has just updated."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small(svr):
    return svr.synth_random_scene(4, 20000, 7, 3)


def test_roundtrip_renders_bit_identically(svr, ctx, small, tmp_path):
    from oracle import svrx
    for deg, arrays in [(3, small), (1, svr.synth_random_scene(9, 5000, 6, 1))]:
        scene = svr.Scene(ctx, arrays)
        path = str(tmp_path / f"s{deg}.svrx")
        scene.save_svrx(path)
        assert open(path, "rb").read() == svrx.encode(arrays)
        back = svr.Scene.load_svrx(ctx, path)
        b = back.arrays
        for name in ("codes", "levels", "corner_index", "density", "sh"):
            assert np.array_equal(getattr(b, name), getattr(arrays, name)), name
        assert b.sh_degree == deg and b.bounds_size == arrays.bounds_size
        cam = svr.ring_camera(1, 0, 24, 24)
        o = svr.RenderOptions(supersample=1.0)
        ra, rb = svr.render(scene, cam, o), svr.render(back, cam, o)
        assert np.array_equal(ra.color, rb.color) and np.array_equal(ra.depth, rb.depth)


def test_empty_scene(svr, ctx, tmp_path):
    empty = svr.SceneArrays(np.zeros(0, np.uint64), np.zeros(0, np.uint8),
                            np.zeros((0, 8), np.uint32), np.zeros(0, np.float32),
                            np.zeros((0, 48), np.float32), 3, (0.0, 0.0, 0.0), 2.0)
    path = str(tmp_path / "e.svrx")
    svr.Scene(ctx, empty).save_svrx(path)
    assert svr.Scene.load_svrx(ctx, path).arrays.n_voxels == 0


def test_rejects_corruption(svr, ctx, small, tmp_path):
    path = str(tmp_path / "s.svrx")
    svr.Scene(ctx, small).save_svrx(path)
    data = bytearray(open(path, "rb").read())

    def corrupt(off, name):
        b = bytearray(data)
        b[off] = (b[off] + 1) % 256
        p = str(tmp_path / name)
        open(p, "wb").write(bytes(b))
        return p

    with pytest.raises(RuntimeError, match="magic"):
        svr.Scene.load_svrx(ctx, corrupt(0, "magic.svrx"))
    with pytest.raises(RuntimeError, match="checksum"):
        svr.Scene.load_svrx(ctx, corrupt(len(data) // 2, "flip.svrx"))
    tiny = str(tmp_path / "tiny.svrx")
    open(tiny, "wb").write(b"SVRX")
    with pytest.raises(RuntimeError):
        svr.Scene.load_svrx(ctx, tiny)
    with pytest.raises(RuntimeError):
        svr.Scene.load_svrx(ctx, str(tmp_path / "absent.svrx"))


def test_rejects_inconsistent_corner_indexing(svr, ctx, small, tmp_path):
    """io.cpp:342-357: a corner that maps to another pool entry than its
    lattice key does elsewhere is refused (file otherwise valid)."""
    from oracle import svrx
    bad = svr.SceneArrays(small.codes, small.levels, small.corner_index.copy(), small.density,
                          small.sh, small.sh_degree, small.bounds_center, small.bounds_size)
    bad.corner_index[0, 7], bad.corner_index[1, 7] = bad.corner_index[1, 7], bad.corner_index[0, 7]
    p = str(tmp_path / "bad.svrx")
    open(p, "wb").write(svrx.encode(bad))
    with pytest.raises(RuntimeError, match="corner indexing|orphaned"):
        svr.Scene.load_svrx(ctx, p)


def test_checkpoint_after_device_training(svr, ctx, small, tmp_path):
    import torch
    from paper_2412_04459_b200.trainer import DeviceTrainer
    scene = svr.Scene(ctx, small)
    tr = DeviceTrainer(svr, ctx, scene, svr.RenderOptions(K=1, supersample=1.0))
    gt = torch.full((32, 32, 3), 0.4, dtype=torch.float32, device="cuda")
    for _ in range(3):
        tr.step(svr.ring_camera(1, 0, 32, 32), gt)
    d, s = tr.params()
    path = str(tmp_path / "t.svrx")
    scene.save_svrx(path)
    back = svr.Scene.load_svrx(ctx, path).arrays
    assert np.array_equal(back.density, d) and np.array_equal(back.sh.reshape(-1), s)
    assert not np.array_equal(back.density, small.density)


def test_save_is_byte_identical_to_reference_and_loads_both_ways(svr, ctx, ref, tmp_path):
    for seed, target, maxlv, deg in [(4, 20000, 7, 3), (9, 5000, 6, 1), (3, 600, 5, 0)]:
        rs = ref.RefScene.generate(seed, target, maxlv, deg)
        a = rs.arrays()
        ours, theirs = str(tmp_path / f"o{seed}.svrx"), str(tmp_path / f"r{seed}.svrx")
        svr.Scene(ctx, a).save_svrx(ours)
        rs.save_checkpoint(theirs)
        assert open(ours, "rb").read() == open(theirs, "rb").read()
        # reference file -> our device loader; our file -> the reference loader
        mine = svr.Scene.load_svrx(ctx, theirs).arrays
        back = ref.RefScene.load_checkpoint(ours).arrays()
        for f in ("codes", "levels", "corner_index", "density", "sh"):
            assert np.array_equal(getattr(mine, f), getattr(a, f)), f
            assert np.array_equal(getattr(back, f), getattr(a, f)), f
        assert tuple(mine.bounds_center) == tuple(back.bounds_center)
        assert mine.bounds_size == back.bounds_size and mine.sh_degree == deg


def test_corrupt_files_rejected_like_the_reference(svr, ctx, ref, small, tmp_path):
    """Every corruption the reference's load_checkpoint refuses, ours refuses
    (and the reverse), on single-byte flips across the header and payload."""
    path = str(tmp_path / "s.svrx")
    svr.Scene(ctx, small).save_svrx(path)
    data = open(path, "rb").read()
    rng = np.random.default_rng(3)
    offs = sorted(set([0, 3, 4, 8, 12, 16, 20, 40, 64] + list(rng.integers(0, len(data), 24))))
    for off in offs:
        b = bytearray(data)
        b[off] ^= 0x5A
        p = str(tmp_path / f"c{off}.svrx")
        open(p, "wb").write(bytes(b))
        ours_ok = theirs_ok = True
        try:
            svr.Scene.load_svrx(ctx, p)
        except RuntimeError:
            ours_ok = False
        try:
            ref.RefScene.load_checkpoint(p)
        except (RuntimeError, ValueError):
            theirs_ok = False
        assert ours_ok == theirs_ok, f"byte {off}: ours {ours_ok}, reference {theirs_ok}"
