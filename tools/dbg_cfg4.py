"""Worst-depth pixel of the cfg4 parity view: per-contribution comparison."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2412_04459_b200 as svr
from oracle import ref
ref.load_ref()
ctx = svr.Context(0, debug=True)
cams = [svr.ring_camera(8, i, 1024, 1024) for i in range(8)]
arrays = svr.synth_unbounded_scene(cams, 7, 5, 2.8, seed=7)
scene = svr.Scene(ctx, arrays); rscene = ref.RefScene.from_arrays(arrays)
view = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cam = svr.ring_camera(256, view, 64, 64, 1.0)
opts = svr.RenderOptions(supersample=1.0, training=True)
out = svr.render(scene, cam, opts)
rf = ref.RefFrame(rscene, cam, opts)
dd = np.abs(out.depth.astype(np.float64) - rf.depth); dd[rf.depth > 1e20] = 0
print("depth err max", dd.max(), "mean", dd.mean(), "mean signed", np.mean((out.depth - rf.depth)[rf.depth < 1e20]))
print("color err", np.abs(out.color - rf.color).max(), "T err", np.abs(out.transmittance - rf.transmittance).max())
py, px = np.unravel_index(np.argmax(dd), dd.shape)
print("worst px", px, py, out.depth[py, px], rf.depth[py, px], "T", out.transmittance[py, px], rf.transmittance[py, px])
pre, cp, ca, cb, pb, pc = out.frame.records()
pre_r, cp_r, ca_r, cb_r, pb_r, pc_r, _ = rf.records()
p = py * 64 + px
s, n = pb[p], pc[p]; sr, nr = pb_r[p], pc_r[p]
print("contribs ours", n, "ref", nr, "same list", np.array_equal(cp[s:s+n], cp_r[sr:sr+nr]))
# double-precision alpha from the scene arrays
codes, levels = arrays.codes, arrays.levels
bc, bs = np.asarray(arrays.bounds_center, np.float64), float(arrays.bounds_size)
def geom(v):
    l = int(levels[v]); c = int(codes[v]) >> (3 * (16 - l)); i = j = k = 0
    for b in range(l):
        i |= ((c >> 2) & 1) << b; j |= ((c >> 1) & 1) << b; k |= (c & 1) << b; c >>= 3
    size = bs * 2.0 ** -l
    return bc - 0.5 * bs + size * (np.array([i, j, k]) + 0.5), size
R = np.asarray(cam.rot, np.float64).reshape(3, 3); pos = np.asarray(cam.pos, np.float64)
d = R @ np.array([(px + 0.5 - cam.cx) / cam.fx, (py + 0.5 - cam.cy) / cam.fy, 1.0])
def explin(x): return x if x > 1.1 else np.exp(x / 1.1 - 1 + np.log(1.1))
def tri(V, q):
    w = [((1 - q[0]) if not (c >> 2) & 1 else q[0]) * ((1 - q[1]) if not (c >> 1) & 1 else q[1]) * ((1 - q[2]) if not c & 1 else q[2]) for c in range(8)]
    return sum(w[c] * V[c] for c in range(8))
def run(cps, A, B):
    T = 1.0; dep = 0.0; rows = []
    for i in range(len(cps)):
        v = pre[cps[i]] if False else None
    return
for label, cps, A, B, prel in [("ours", cp[s:s+n], ca[s:s+n], cb[s:s+n], pre), ("ref", cp_r[sr:sr+nr], ca_r[sr:sr+nr], cb_r[sr:sr+nr], pre_r)]:
    T = 1.0; dep = 0.0
    for i in range(len(cps)):
        vid = prel[cps[i]]
        c, size = geom(vid)
        V = arrays.density[arrays.corner_index[vid]].astype(np.float64)
        a, b = A[i], B[i]
        l = (b - a) * np.linalg.norm(d)
        t = a + 0.5 * (b - a)
        q = (pos + t * d - (c - 0.5 * size)) / size
        al = 1 - np.exp(-l * explin(tri(V, q)))
        dep += T * al * t; T *= 1 - al
    print(label, "double recompute depth", dep, "T", T)
print("seg diff (ours-ref) per contrib:")
m = min(n, nr)
for i in range(m):
    vid = pre[cp[s+i]]; c, size = geom(vid)
    print(i, vid, "size %.3e" % size, "a %.9f b %.9f" % (ca_r[sr+i], cb_r[sr+i]), "da %.2e db %.2e dseg/seg %.2e" % (ca[s+i]-ca_r[sr+i], cb[s+i]-cb_r[sr+i], ((cb[s+i]-ca[s+i])-(cb_r[sr+i]-ca_r[sr+i]))/max(1e-30,(cb_r[sr+i]-ca_r[sr+i]))))
