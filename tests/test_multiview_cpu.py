"""world_size-2 gloo tests (CPU) of the multi-GPU host logic: view sharding
covers every view exactly once, and the flat-buffer all-reduce of per-rank
gradients equals the single-process sum of per-view render_backward
gradients (the oracle of SURVEY §8(e)); per-view gradients come from the C
oracle here, from the CUDA kernels on the GPU box."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_04459_b200.multiview import allreduce_flat, flat_layout, shard_views


def sum_gradients_reference(per_view_grads):
    """Oracle for the all-reduce: element-wise sum of per-view gradients."""
    return {k: np.sum([np.asarray(g[k], np.float64).reshape(-1) for g in per_view_grads], axis=0)
            for k in ("density", "sh", "priority")}


def test_shard_views_partition():
    for n, w in [(256, 1), (256, 2), (256, 8), (10, 4), (3, 8)]:
        owned = [shard_views(n, r, w) for r in range(w)]
        flat = sorted(v for o in owned for v in o)
        assert flat == list(range(n))
        assert max(map(len, owned)) - min(map(len, owned)) <= 1
    with pytest.raises(ValueError):
        shard_views(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _per_view_grads(view):
    import paper_2412_04459_b200 as svr
    from oracle import port
    a = svr.synth_random_scene(11, 900, 5, 1)
    cam = svr.ring_camera(4, view, 24, 20)
    opts = svr.RenderOptions(K=1, supersample=1.0, training=True)
    r = port.render(a, cam, svr.RenderOptions(K=1, supersample=1.0))
    gt = np.random.default_rng(100 + view).uniform(0, 1, r["color"].shape)
    d_color = np.sign(r["color"] - gt) / r["color"].size
    return a, port.backward(a, cam, opts, d_color)


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a = None
    n_pool = n_sh = 0
    flat = None
    for v in shard_views(4, rank, world):
        a, g = _per_view_grads(v)
        n_pool, n_sh = a.n_pool, a.n_voxels * a.sh_stride
        d0, s0, p0, total = flat_layout(n_pool, n_sh, a.n_voxels)
        if flat is None:
            flat = torch.zeros(total, dtype=torch.float64)
        flat[d0:d0 + n_pool] += torch.from_numpy(g["density"])
        flat[s0:s0 + n_sh] += torch.from_numpy(g["sh"].reshape(-1))
        flat[p0:p0 + a.n_voxels] += torch.from_numpy(g["priority"])
    allreduce_flat(flat)
    if rank == 0:
        np.save(out_path, flat.numpy())
    dist.destroy_process_group()


def test_sharded_gradient_allreduce_equals_sum(tmp_path):
    out = str(tmp_path / "flat.npy")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    flat = np.load(out)
    grads = [_per_view_grads(v)[1] for v in range(4)]
    a = _per_view_grads(0)[0]
    ref = sum_gradients_reference(grads)
    d0, s0, p0, total = flat_layout(a.n_pool, a.n_voxels * a.sh_stride, a.n_voxels)
    assert np.allclose(flat[d0:d0 + a.n_pool], ref["density"], rtol=1e-12, atol=1e-15)
    assert np.allclose(flat[s0:s0 + a.n_voxels * a.sh_stride], ref["sh"], rtol=1e-12, atol=1e-15)
    assert np.allclose(flat[p0:p0 + a.n_voxels], ref["priority"], rtol=1e-12, atol=1e-15)
    assert np.abs(ref["density"]).max() > 0
