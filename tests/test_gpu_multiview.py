"""The config-5 training step with two ranks: two processes
share the one GPU of the test box over gloo (a real 2-GPU run would use
NCCL over NVLink; the host logic and the flat [density | SH | priority]
all-reduce are the same). Each rank runs ShardedTrainer.step over its views
of a 4-view batch; the all-reduced gradient must equal the single-process
sum of the 4 views and the sum of the reference's per-view train steps
(rel 1e-3)."""
import os
import socket

import numpy as np
import pytest

from conftest import grad_close, untie_gt

pytestmark = pytest.mark.gpu

VIEWS, RES = 4, 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(svr, ctx):
    arrays = svr.synth_random_scene(2024, 65536, 7, 3)
    scene = svr.Scene(ctx, arrays)
    cams = [svr.ring_camera(VIEWS, v, RES, RES) for v in range(VIEWS)]
    opts = svr.RenderOptions(K=1, supersample=1.0, training=True)
    return arrays, scene, cams, opts


def _worker(rank, world, port, gt_path, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_2412_04459_b200 as svr
    from paper_2412_04459_b200.multiview import ShardedTrainer, shard_views
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ctx = svr.Context(0)
    arrays, scene, cams, opts = _setup(svr, ctx)
    gts = list(np.load(gt_path))
    tr = ShardedTrainer(ctx, scene, cams, gts, opts)
    loss = tr.step(shard_views(VIEWS, rank, world))  # all-reduced in place
    g = tr.gradients()
    lt = torch.tensor([loss], dtype=torch.float64)
    dist.all_reduce(lt)
    if rank == 0:
        np.savez(out_path, loss=lt.item(), **g)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_allreduce_matches_single_process_and_reference(svr, ref, tmp_path):
    import torch.multiprocessing as mp

    from paper_2412_04459_b200.multiview import ShardedTrainer
    ctx = svr.Context(0)
    arrays, scene, cams, opts = _setup(svr, ctx)
    rscene = ref.RefScene.from_arrays(arrays)
    rng = np.random.default_rng(5)
    gts = []
    for c in cams:
        g = rng.uniform(0, 1, (RES, RES, 3))
        gts.append(untie_gt(g, svr.render(scene, c, opts).color).astype(np.float32))
    gt_path = str(tmp_path / "gts.npy")
    np.save(gt_path, np.stack(gts))
    out = str(tmp_path / "reduced.npz")
    mp.start_processes(_worker, args=(2, _free_port(), gt_path, out), nprocs=2, join=True,
                       start_method="spawn")
    red = np.load(out)

    single = ShardedTrainer(ctx, scene, cams, gts, opts)
    loss1 = single.step(list(range(VIEWS)), reduce=False)
    g1 = single.gradients()
    per_view = [ref.ref_train_step_l1(rscene, c, opts, g.astype(np.float64), arrays.n_pool,
                                      arrays.n_voxels * arrays.sh_stride, arrays.n_voxels)
                for c, g in zip(cams, gts)]
    assert abs(float(red["loss"]) - loss1) <= 1e-5 * max(1.0, abs(loss1))
    assert abs(loss1 - sum(p[0] for p in per_view)) <= 1e-5 * VIEWS
    for k, name in [(2, "density"), (3, "sh"), (4, "priority")]:
        theirs = np.sum([p[k] for p in per_view], axis=0)
        for label, ours in [("2-rank", red[name]), ("1-rank", g1[name])]:
            nbad, worst = grad_close(ours, theirs)
            assert nbad == 0, f"{label} {name}: {nbad} out of tolerance (worst {worst:.3e})"
        # the two ranks' partial sums differ from one accumulation only by fp32
        # reassociation (and float atomics are order-nondeterministic run to
        # run), so they agree by the same rule
        nbad, _ = grad_close(red[name], g1[name])
        assert nbad == 0, name
    assert np.abs(red["density"]).max() > 0


def test_c_abi_batch_step_and_nccl_allreduce(svr, ref):
    """svr_train_batch_l1 (the C-ABI sharded step a C++ caller uses) equals
    ShardedTrainer's torch-side accumulation; on a one-rank NCCL communicator
    svr_comm_allreduce_gradients is the identity and svr_comm_check is clean."""
    import ctypes as C

    import torch

    from paper_2412_04459_b200.multiview import NcclComm, ShardedTrainer
    ctx = svr.Context(0)
    arrays, scene, cams, opts = _setup(svr, ctx)
    rng = np.random.default_rng(9)
    gts = [rng.uniform(0, 1, (RES, RES, 3)).astype(np.float32) for _ in cams]
    comm = NcclComm(ctx, NcclComm.make_id(), 0, 1)
    a = ShardedTrainer(ctx, scene, cams, gts, opts)
    la = a.step([0, 1, 2, 3], reduce=False)
    ga = a.gradients()
    b = ShardedTrainer(ctx, scene, cams, gts, opts, comm=comm)
    lb = b.step([0, 1, 2, 3])
    gb = b.gradients()
    assert abs(la - lb) <= 1e-6 * max(1.0, abs(la))
    for k in ("density", "sh", "priority"):  # fp32 atomics: run-to-run reassociation only
        nbad, _ = grad_close(gb[k], ga[k])
        assert nbad == 0, k
    # the NCCL all-reduce itself, one rank: identity, in place
    before = b.flat.clone()
    g = svr.svr_gradients()
    g.density, g.sh, g.priority, g.on_device = (b.density_grad.data_ptr(), b.sh_grad.data_ptr(),
                                                b.priority.data_ptr(), 1)
    lib = svr.load_library()
    svr._check(lib.svr_comm_allreduce_gradients(comm.h, C.byref(g), b.n_pool, b.n_sh, b.n_vox))
    ctx.synchronize()
    assert torch.equal(before, b.flat)
    comm.check()
    # an empty batch contributes zeros
    assert b.step([]) == 0.0 and float(b.flat.abs().max()) == 0.0
    comm.close()
