"""Generates the golden fixtures of tests/golden/ from the UNMODIFIED reference.

Run in a container that has /root/reference (oracle/_ref/libsvr_ref.so is
built from it by `make -C oracle ref`):   python tests/golden/make_golden.py

Fixture = one small scene from generator G (fully determined by its seed, so
only the seed and a checksum of the arrays are stored), two cameras/option
sets, and the reference's outputs on them: tile masks, per-voxel projection,
emitted and sorted entries, the five images, and render_backward gradients
for an L1 upstream. Every array is exactly what proj/src/raster.cpp computes.
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2412_04459_b200 as svr  # noqa: E402  (generator + structs only)
from oracle import ref  # noqa: E402

SCENE = dict(seed=2024, target=1500, max_level=6, sh_degree=2)
CASES = [
    dict(name="ss1_K2", view=(2, 0, 64, 48), ss=1.0, K=2, bg=(0.1, 0.2, 0.3)),
    dict(name="ss15_K1", view=(2, 1, 40, 30), ss=1.5, K=1, bg=(0.0, 0.0, 0.0)),
]


def scene_digest(a) -> str:
    h = hashlib.sha256()
    for x in (a.codes, a.levels, a.corner_index, a.density, a.sh):
        h.update(np.ascontiguousarray(x).tobytes())
    return h.hexdigest()


def main():
    a = svr.synth_random_scene(**SCENE)
    rs = ref.RefScene.generate(**SCENE)
    ra = rs.arrays()
    assert scene_digest(a) == scene_digest(ra), "generator G differs from the reference build"
    out = {"scene_digest": np.array(scene_digest(a)), "scene_params": np.array(
        [SCENE["seed"], SCENE["target"], SCENE["max_level"], SCENE["sh_degree"]])}
    for c in CASES:
        n = c["name"]
        cam = svr.ring_camera(*c["view"])
        opts = svr.RenderOptions(K=c["K"], supersample=c["ss"], background=c["bg"])
        scam = ref.ref_scaled_camera(cam, c["ss"])
        out[f"{n}/camera"] = np.concatenate([[cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy],
                                             np.asarray(cam.rot).reshape(9), cam.pos])
        out[f"{n}/opts"] = np.array([c["K"], c["ss"], *c["bg"]])
        out[f"{n}/tile_masks"] = ref.ref_tile_masks(scam)
        vis, aabb, rect = ref.ref_project(rs, scam, a.n_voxels)
        out[f"{n}/visible"], out[f"{n}/aabb"], out[f"{n}/rect"] = vis, aabb, rect
        out[f"{n}/entry_keys"], out[f"{n}/entry_values"] = ref.ref_entries(rs, scam, False)
        out[f"{n}/sorted_keys"], out[f"{n}/sorted_values"] = ref.ref_entries(rs, scam, True)
        r = ref.ref_render(rs, cam, opts)
        for k in ("color", "depth", "median_depth", "normal", "transmittance"):
            out[f"{n}/{k}"] = r[k]
        gt = np.random.default_rng(17).uniform(0, 1, r["color"].shape)
        topts = svr.RenderOptions(K=c["K"], supersample=c["ss"], background=c["bg"], training=True)
        loss, dcol, gd, gs, gp = ref.ref_train_step_l1(rs, cam, topts, gt, a.n_pool,
                                                       a.n_voxels * a.sh_stride, a.n_voxels)
        out[f"{n}/gt"] = gt
        out[f"{n}/l1_loss"] = np.array(loss)
        out[f"{n}/d_color"] = dcol
        out[f"{n}/g_density"], out[f"{n}/g_sh"], out[f"{n}/g_priority"] = gd, gs, gp
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_small.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
