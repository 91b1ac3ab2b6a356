import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2412_04459_b200 as svr
from oracle import ref
from conftest import look_at_origin, grad_close
ref.load_ref()
ctx = svr.Context(0, debug=True)
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
_, dcol, gd, gs, gp = ref.ref_train_step_l1(rs, cam, opts, gt, a.n_pool, a.n_voxels * a.sh_stride, a.n_voxels)
out = svr.render(scene, cam, opts)
r = ref.ref_render(rs, cam, opts)
for k in ["color", "depth", "transmittance", "normal"]:
    print(k, np.max(np.abs(getattr(out, k) - r[k])))
g = svr.render_backward(scene, out.frame, d_color=dcol)
print("sh ours", g.sh.reshape(2, -1)[:, :3]); print("sh ref", gs.reshape(2, -1)[:, :3])
print("density", grad_close(g.density, gd), "sh", grad_close(g.sh, gs), "prio", grad_close(g.priority, gp))
print(g.priority, gp)
d = np.abs(out.depth - r["depth"]); i = np.unravel_index(np.argmax(d), d.shape)
print("worst depth px", i, out.depth[i], r["depth"][i], "T", out.transmittance[i], r["transmittance"][i])
print("sh full ours", g.sh.reshape(2, -1)); print("sh full ref", gs.reshape(2, -1))
