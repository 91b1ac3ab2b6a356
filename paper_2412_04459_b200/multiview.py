"""Multi-GPU paths of the rasterizer: the two partitioned workloads of
SURVEY §8(e).

* View-sharded rendering (config 4): every rank holds a replica of the scene
  and renders its own subset of the views; no collective on the data path.
* View-batch training step (config 5): every rank runs forward -> L1 ->
  backward for its views into ONE flat gradient buffer
  [density (P) | SH (N*stride) | priority (N)] and the ranks sum it with a
  single in-place all-reduce (NCCL over NVLink on B200s; gloo in the tests),
  so every replica sees the same gradients and the same subdivision
  priorities.

One process per GPU (torch.distributed for the plumbing). The reference has
no distributed code; the sum of per-view `render_backward` gradients is the
oracle (tests/test_multiview_cpu.py: host logic over gloo on CPU;
tests/test_gpu_multiview.py: two ranks sharing one GPU over gloo against the
single-process sum and the reference; tests/test_gpu_fullsize.py: the
config-5 batch sum against the reference).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np


def shard_views(n_views: int, rank: int, world: int) -> List[int]:
    """Views owned by `rank`: rank, rank+world, ... (balanced to within one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    return list(range(rank, n_views, world))


def flat_layout(n_pool: int, n_sh: int, n_vox: int = 0, align: int = 64):
    """Offsets (in floats) of the density, SH and priority gradients in the
    flat buffer, and its total length: (0, sh_off, prio_off, total)."""
    up = lambda x: (x + align - 1) // align * align  # noqa: E731
    sh_off = up(n_pool)
    prio_off = up(sh_off + n_sh)
    return 0, sh_off, prio_off, prio_off + n_vox


class NcclComm:
    """svr_comm (include/svr_b200.h): the library's own NCCL communicator for
    the C-ABI training step (svr_train_batch_l1), one per rank. `unique_id`
    comes from rank 0's NcclComm.make_id(), handed to the others by the
    caller (e.g. a torch.distributed broadcast)."""

    def __init__(self, ctx, unique_id: bytes, rank: int, world: int):
        import paper_2412_04459_b200 as svr
        self.svr, self.ctx = svr, ctx
        lib = svr.load_library()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        svr._check(lib.svr_comm_create(ctx.h, buf, rank, world, C.byref(h)))
        self.h, self.rank, self.world = h, rank, world

    @staticmethod
    def make_id() -> bytes:
        import paper_2412_04459_b200 as svr
        buf = (C.c_uint8 * 128)()
        svr._check(svr.load_library().svr_comm_unique_id(buf))
        return bytes(buf)

    def register(self, tensor) -> None:
        self.svr._check(self.svr.load_library().svr_comm_register(
            self.h, C.c_void_p(tensor.data_ptr()), C.c_size_t(tensor.numel() * tensor.element_size())))

    def check(self) -> None:
        self.svr._check(self.svr.load_library().svr_comm_check(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            self.svr.load_library().svr_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def allreduce_flat(buf, group=None) -> None:
    """Sums the flat gradient buffer over all ranks, in place (one collective)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)


class ShardedTrainer:
    """Config-5 training step on this rank's GPU.

    `step(view_ids)` renders each view with training records, applies the L1
    loss against its ground truth and accumulates render_backward into the
    flat device gradient buffer, then all-reduces it across ranks.
    """

    def __init__(self, ctx, scene, cameras: Sequence, gts: Sequence, opts, group=None,
                 comm: Optional["NcclComm"] = None):
        import torch

        import paper_2412_04459_b200 as svr
        self.svr = svr
        self.ctx, self.scene, self.cams, self.opts, self.group = ctx, scene, cameras, opts, group
        self.comm = comm  # NcclComm: the whole step through svr_train_batch_l1
        dev = torch.device("cuda", ctx.device)
        self.gts = [g if isinstance(g, torch.Tensor) else
                    torch.tensor(np.asarray(g), dtype=torch.float32, device=dev) for g in gts]
        a = scene.arrays
        self.n_pool, self.n_sh, self.n_vox = a.n_pool, a.n_voxels * a.sh_stride, a.n_voxels
        d0, s0, p0, total = flat_layout(self.n_pool, self.n_sh, self.n_vox)
        self.flat = torch.zeros(total, dtype=torch.float32, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.density_grad = self.flat[d0:d0 + self.n_pool]
        self.sh_grad = self.flat[s0:s0 + self.n_sh]
        self.priority = self.flat[p0:p0 + self.n_vox]
        self.frame = svr.Frame(ctx)
        self.stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
        if comm is not None:
            comm.register(self.flat)

    def step(self, view_ids: Sequence[int], reduce: bool = True, lazy: bool = False):
        """One batch: forward -> L1 -> backward of `view_ids` accumulated into
        the flat gradient, all-reduced across ranks when `reduce`. Returns the
        summed loss as a float, or (lazy) as a one-element device tensor the
        caller reads back when it needs it (pipelined loops)."""
        import torch
        svr = self.svr
        lib = svr.load_library()
        g = svr.svr_gradients()
        g.density, g.sh = self.density_grad.data_ptr(), self.sh_grad.data_ptr()
        g.priority, g.on_device = self.priority.data_ptr(), 1
        # the library stream runs after the caller's pending work (ground
        # truths, the flat buffer) without a host round trip
        self.stream.wait_stream(torch.cuda.current_stream())
        if self.comm is not None:  # one C-ABI call: views, loss sum, NCCL all-reduce
            n = len(view_ids)
            cams = (svr.svr_camera * max(n, 1))(*[self.cams[v].to_c() for v in view_ids])
            gts = (C.c_void_p * max(n, 1))(*[self.gts[v].data_ptr() for v in view_ids])
            o = self.opts.to_c()
            svr._check(lib.svr_train_batch_l1(self.ctx.h, self.scene.h, cams, gts, n, C.byref(o),
                                              self.frame.h, C.byref(g),
                                              self.comm.h if reduce else None,
                                              C.c_void_p(self.loss.data_ptr())))
            torch.cuda.current_stream().wait_stream(self.stream)
            return self.loss.clone() if lazy else float(self.loss.item())
        if not view_ids:  # no view on this rank: contribute zeros to the sum
            with torch.cuda.stream(self.stream):
                self.flat.zero_()
        total = 0.0
        for n, v in enumerate(view_ids):
            c, o = self.cams[v].to_c(), self.opts.to_c()
            svr._check(lib.svr_train_step_l1(self.ctx.h, self.scene.h, C.byref(c), C.byref(o),
                                             C.c_void_p(self.gts[v].data_ptr()), self.frame.h,
                                             C.byref(g), int(n > 0),  # first view overwrites
                                             C.c_void_p(self.loss.data_ptr())))
            with torch.cuda.stream(self.stream):
                total += self.loss  # device scalar, read once below
        with torch.cuda.stream(self.stream):
            loss_t = total if isinstance(total, torch.Tensor) else torch.zeros(1, device=self.flat.device)
        torch.cuda.current_stream().wait_stream(self.stream)
        if reduce:
            allreduce_flat(self.flat, self.group)
        return loss_t if lazy else float(loss_t.item())

    def gradients(self) -> dict:
        """The (reduced) gradients of the last step as host float32 arrays."""
        import torch
        torch.cuda.current_stream().wait_stream(self.stream)
        return {"density": self.density_grad.cpu().numpy(), "sh": self.sh_grad.cpu().numpy(),
                "priority": self.priority.cpu().numpy()}
