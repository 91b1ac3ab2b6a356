#!/usr/bin/env python
"""Benchmark of the B200 sparse-voxel rasterizer (BASELINE.json metric).

Default workload (the driver's bench line) is config 2:
metric : FPS @1024x1024 on the 1M-voxel scene, reported as frames/s (whole
         job, all ranks) plus Mrays/s and the HBM roofline of the dominant
         kernel.
step   : one forward render (svr::render path: preprocess -> duplicate ->
         onesweep sort -> tile ranges -> composite) of one 1024x1024 view per
         GPU. Views come from ring_cameras(256, ...) (view 0 is exactly
         config 2's camera); rank r renders views r, r+N, r+2N, ... (weak
         scaling, no collective on the data path).
value  : device time, CUDA events on the library's stream around each step,
         L2 flushed (256 MiB write) before every timed step, max over ranks.
e2e    : the same step through the C ABI with host buffers: camera in, all
         five output images (37.7 MB) copied back to pinned host memory every
         step, wall clock, max over ranks.

Other SURVEY §8(d) workloads (--workload; bench lines for profiles/, the
driver runs the default):
  cfg3  training step at 800x800 on the 1M scene: forward (with records) ->
        L1 against a U(0,1) image -> render_backward to density/SH.
  cfg4  8M-voxel init_unbounded scene, 1024^2 views of ring_cameras(256, ...,
        radius 1.0) sharded by view.
  cfg5  cfg4 scene, training step on a batch of 4 views per GPU with one
        in-place all-reduce of the flat [density | SH | priority] gradient
        (the library's NCCL communicator, svr_train_batch_l1).

--impl reference : the reference's own CPU implementation (oracle/_ref,
         compiled unmodified) on this host's cores, same metric/config.

Run: python bench.py [--gpus N --steps K --warmup W --workload cfgX]; N>1
under torchrun.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_VIEWS = 256
G_SCENE = dict(seed=7, target=1 << 20, max_level=9, sh_degree=3)
U_SCENE = dict(init_level=7, shell_levels=5, bg_ratio=2.8, seed=7, sh_degree=3)
WORKLOADS = {
    "cfg2": dict(kind="render", scene="G", res=1024, dist=1.3, batch=1,
                 metric="FPS @1024x1024 (1M voxels)", unit="frames/s",
                 desc="cfg2: generator G(seed 7, 2^20, max level 9) -> 1,048,573 leaf voxels "
                      "(L3-9), SH degree 3; 1024x1024, supersample 1.0, K=1, t_threshold 1e-4, "
                      "bg 0; views ring_cameras(256, 1024, 1024, 1.3, 55 deg), rank r renders "
                      "views r, r+N, ..."),
    "cfg3": dict(kind="train", scene="G", res=800, dist=1.3, batch=1,
                 metric="training steps/s @800x800 (1M voxels)", unit="steps/s",
                 desc="cfg3: cfg2 scene, ring_cameras(1, 800, 800, 1.3, 55 deg)[0], gt U(0,1) "
                      "seed 17; forward with records -> L1 -> render_backward to density, SH "
                      "(and priority), K=1, supersample 1.0"),
    "cfg3i": dict(kind="iter", scene="G", res=800, dist=1.3, batch=1,
                  metric="training iterations/s @800x800 (1M voxels)", unit="iters/s",
                  desc="cfg3 scene and view, one full optim::train iteration on the device "
                       "(trainer.DeviceTrainer): render with records -> MSE + 0.02 SSIM -> ray "
                       "losses (lambda_T 0.01, lambda_dist 0.1, lambda_R 0.01) -> render_backward "
                       "-> Adam on the density and SH pools (optim.cpp:433-495 minus adaptation)"),
    "cfg4": dict(kind="render", scene="U", res=1024, dist=1.0, batch=1,
                 metric="FPS @1024x1024 (8M voxels, 256 views)", unit="frames/s",
                 desc="cfg4: init_unbounded(ring_cameras(8, 1024, 1024, 1.3, 55 deg), init_level "
                      "7, shell_levels 5, bg_ratio 2.8) -> 7,824,544 voxels (L2-16), parameters "
                      "as G (seed 7); 1024x1024 views of ring_cameras(256, 1024, 1024, 1.0, 55 "
                      "deg), rank r renders views r, r+N, ..."),
    "cfg5": dict(kind="train", scene="U", res=1024, dist=1.0, batch=4,
                 metric="training views/s @1024x1024 (8M voxels)", unit="views/s",
                 desc="cfg5: cfg4 scene; per GPU a batch of 4 views of ring_cameras(256, 1024, "
                      "1024, 1.0, 55 deg) (rank r: views 4(r + N i) .. +3), gt U(0,1) seed "
                      "17+view; forward -> L1 -> backward into one flat [density | SH] buffer, "
                      "in-place all-reduce (NCCL) across ranks"),
}
# the driver's metric/config (BASELINE.json) is config 2's
METRIC = WORKLOADS["cfg2"]["metric"]
UNIT = WORKLOADS["cfg2"]["unit"]
WORKLOAD = WORKLOADS["cfg2"]["desc"]


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--supersample", type=float, default=1.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-dropin", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=100)
    p.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=1)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ roofline
def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def stage_bytes(stage, d):
    """Algorithmic bytes per launch. d: n_vox, n_pool, n_vis,
    E, R, ntiles, stride, npass, contribs."""
    if stage == "composite":
        # the 96-B record of each visible voxel read once, the
        # 4-B sorted value of each entry, 8 B of range per tile, 9 fp32
        # output channels per pixel (re-reads of a record by other tiles are
        # cache traffic, not algorithmic bytes)
        return d["n_vis"] * 96 + d["E"] * 4 + d["ntiles"] * 8 + d["R"] * 36
    if stage == "preprocess":
        return d["n_vox"] * (8 + 16 + 4) + 4 * d["n_pool"] + d["n_vis"] * (32 + 4 * d["stride"] + 96)
    if stage == "sort":
        return d["npass"] * d["E"] * 16
    if stage == "duplicate":  # rank-ordered: pair counts (8n u32) + order/rect per live pair + keys
        return d["n_vox"] * 8 * 4 + d["n_vis"] * (4 + 16) + d["E"] * 8
    if stage == "scan":  # zero + scatter the pair counts, reduce them
        return d["n_vox"] * (8 * 4 + 4 + 8 * 4) + d["n_vis"] * (16 + 8)
    if stage == "backward":
        return (d["E"] * 4 + d["n_vis"] * (96 + 32 + 28) + d["contribs"] * 8 + d["R"] * 20
                + 4 * d["n_pool"])
    if stage == "epilogue":
        return d["n_vox"] * 16 + d["n_vis"] * (8 + 8 * d["stride"] + 24 + 32 + 32)
    return None


def traffic_from_profiles(stage, workload, npass=1):
    """Measured DRAM bytes per launch of `stage` for this workload, from the
    committed ncu summary (profiles/ncu_traffic.json, tools/summarize_ncu.py);
    None when that workload was not captured."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            t = json.load(fh).get(workload, {})
    except (OSError, ValueError, AttributeError):
        return None
    if stage == "sort":
        return t["sort_pass"] * npass if "sort_pass" in t else None
    return t.get(stage)


def make_scene_arrays(svr, w):
    if w["scene"] == "G":
        return svr.synth_random_scene(**G_SCENE)
    cams = [svr.ring_camera(8, i, 1024, 1024) for i in range(8)]
    return svr.synth_unbounded_scene(cams, **U_SCENE)


def view_ids(w, rank, world, i):
    """Views of step i on `rank` (view-sharded, `batch` views per step).
    cfg3 trains on its single view; cfg5 cycles through 4 batches per rank
    (16 ground-truth images resident per GPU)."""
    if w["kind"] in ("train", "iter") and w["scene"] == "G":
        return [0] * w["batch"]
    b = w["batch"]
    first = b * (rank + world * (i % 4 if w["kind"] == "train" else i))
    return [(first + k) % N_VIEWS for k in range(b)]


def make_camera(ring, w, v):
    """View v of workload w; `ring` is ring_cameras (the product's
    svr.ring_camera, or the reference's own ref.ref_ring_camera in the
    reference arm — bit-identical poses, tests/test_abi_cpu.py)."""
    if w["kind"] in ("train", "iter") and w["scene"] == "G":
        return ring(1, 0, w["res"], w["res"], w["dist"])  # cfg3's single view
    return ring(N_VIEWS, v, w["res"], w["res"], w["dist"])


def make_gt(w, v):
    seed = 17 if w["scene"] == "G" else 17 + v
    return np.random.default_rng(seed).uniform(0, 1, (w["res"], w["res"], 3)).astype(np.float32)


def bench_config(w, n_voxels, supersample):
    """The `config` object, identical in both arms (run-specific details go
    under the line's `run` key)."""
    return {"workload": w["desc"], "voxels": int(n_voxels), "resolution": f"{w['res']}x{w['res']}",
            "supersample": supersample, "K": 1, "sh_degree": 3,
            "l2": "GPU arm: L2 flushed (256 MiB write) before every timed step"}


# ------------------------------------------------------------------ reference (CPU)
# This arm never imports paper_2412_04459_b200: the scene, the cameras and the
# options come from the unmodified reference (oracle/_ref: RefScene.generate /
# RefScene.unbounded = init_unbounded, ring_cameras) and oracle/abi.py.
# TrainConfig defaults one iteration uses (optim.hpp:39-60).
TRAIN_DEFAULTS = dict(lr_density=0.025, lr_sh0=0.01, lr_sh_rest=0.00025, lambda_ssim=0.02,
                      lambda_T=0.01, lambda_dist=0.1, lambda_R=0.01)


def ref_scene(ref, w):
    if w["scene"] == "G":
        g = G_SCENE
        return ref.RefScene.generate(g["seed"], g["target"], g["max_level"], g["sh_degree"])
    u = U_SCENE
    cams = [ref.ref_ring_camera(8, i, 1024, 1024) for i in range(8)]
    return ref.RefScene.unbounded(cams, u["init_level"], u["shell_levels"], u["bg_ratio"],
                                  u["seed"], u["sh_degree"])


def band_cameras(cam, threads, rows=None):
    """Horizontal bands of `cam` (each a full camera with shifted cy)."""
    rows = rows or max(16, ((cam.height + threads - 1) // threads + 15) // 16 * 16)
    out = []
    for y0 in range(0, cam.height, rows):
        h = min(rows, cam.height - y0)
        out.append(type(cam)(cam.width, h, cam.fx, cam.fy, cam.cx, cam.cy - y0, cam.rot, cam.pos))
    return out


def reference_step_time(ref, rscene, sizes, w, cam, opts, threads, gt=None, frac=1.0):
    """One step of workload w through the reference's own svr::render (and,
    for training, its L1 + render_backward) split into row bands rendered
    concurrently (the reference API is reentrant; ctypes releases the GIL).
    frac < 1 renders only that fraction of the bands (evenly spread) and
    scales the time. sizes = (n_voxels, n_pool, sh_stride). Returns seconds
    per full step."""
    bands = band_cameras(cam, threads)
    if frac < 1.0:
        keep = max(1, int(round(len(bands) * frac)))
        idx = np.linspace(0, len(bands) - 1, keep).round().astype(int)
        scale = len(bands) / keep
        bands = [bands[i] for i in sorted(set(idx))]
    else:
        scale = 1.0
    n_vox, n_pool, stride = sizes

    def one(c):
        if w["kind"] == "render":
            ref.ref_render(rscene, c, opts)
        else:
            y0 = int(round(cam.cy - c.cy))
            g = gt[y0:y0 + c.height]
            ref.ref_train_step_l1(rscene, c, opts, g, n_pool, n_vox * stride, n_vox)

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=min(threads, len(bands))) as ex:
        list(ex.map(one, bands))
    return (time.perf_counter() - t0) * scale


CPU_FRACTION = {"cfg2": 1.0, "cfg3": 1.0, "cfg3i": 1.0, "cfg4": 1.0 / 16, "cfg5": 1.0 / 16}


def reference_iteration_time(ref, rscene, params, cam, opts, gt):
    """One optim::train iteration (render -> MSE + SSIM -> ray losses ->
    backward -> Adam on both pools) through the unmodified reference, one
    thread (SSIM windows and the pool-wide Adam do not split into bands).
    params = (density, sh, sh_stride) of the scene."""
    density, sh, stride = params
    n_vox = sh.size // stride
    t = TRAIN_DEFAULTS
    t0 = time.perf_counter()
    _, gd, gs, _ = ref.ref_train_iteration_grads(rscene, cam, opts, gt, t["lambda_ssim"],
                                                 t["lambda_T"], t["lambda_dist"], t["lambda_R"],
                                                 density.size, sh.size, n_vox)
    ref.ref_adam_step(density, gd, np.zeros(gd.size), np.zeros(gd.size), 0, t["lr_density"])
    ref.ref_adam_step(sh.reshape(-1), gs, np.zeros(gs.size), np.zeros(gs.size), 0, t["lr_sh0"],
                      t["lr_sh_rest"], stride, 3)
    return time.perf_counter() - t0


def cpu_sample_text(w, name, cores):
    frac = CPU_FRACTION[name]
    if w["kind"] == "iter":
        return (f"one {w['res']}x{w['res']} {name} training iteration (render, MSE + SSIM, ray "
                f"losses, render_backward, Adam on both pools) through the unmodified reference "
                f"(oracle/_ref), single-threaded")
    what = "render" if w["kind"] == "render" else "train step (render + L1 + render_backward)"
    part = "the full view" if frac >= 1.0 else f"{frac:.4g} of the view's row bands (evenly spread), time scaled up"
    return (f"one {w['res']}x{w['res']} {name} {what} through the unmodified reference "
            f"(oracle/_ref) split into row bands on {cores} threads; {part}")


def cpu_step_fn(ref, rscene, w, name, opts, ring, cores):
    """step(i) -> seconds of the reference's CPU path for step i."""
    n_vox, n_pool, deg = rscene.sizes()
    stride = 3 * (deg + 1) ** 2
    params = None
    if w["kind"] == "iter":
        a = rscene.arrays()
        params = (a.density, a.sh, stride)

    def step(i):
        t = 0.0
        for v in view_ids(w, 0, 1, i):
            cam = make_camera(ring, w, v)
            if w["kind"] == "iter":
                t += reference_iteration_time(ref, rscene, params, cam, opts, make_gt(w, v))
                continue
            t += reference_step_time(ref, rscene, (n_vox, n_pool, stride), w, cam, opts, cores,
                                     make_gt(w, v) if w["kind"] == "train" else None,
                                     CPU_FRACTION[name])
        return t
    return step


def run_reference(args, rank):
    if rank != 0:
        return
    from oracle import abi, ref
    w = WORKLOADS[args.workload]
    cores = 1 if w["kind"] == "iter" else host_cores()
    rscene = ref_scene(ref, w)
    opts = abi.RenderOptions(K=1, supersample=args.supersample, training=w["kind"] != "render")
    step = cpu_step_fn(ref, rscene, w, args.workload, opts, ref.ref_ring_camera, cores)
    for i in range(args.warmup):
        step(i)
    total = sum(step(i) for i in range(args.steps))
    units = args.steps * w["batch"]
    val = units / total
    sw = int(np.ceil(args.supersample * w["res"]))
    line = {
        "impl": "reference", "metric": w["metric"], "value": val, "unit": w["unit"],
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "mrays_per_s": val * sw * sw / 1e6,
        "config": bench_config(w, rscene.sizes()[0], args.supersample),
        "run": {"parallelism": f"{cores} CPU thread(s), row bands of each view"},
        "cpu_baseline": {"value": val, "unit": w["unit"], "cores": cores, "kind": "reference",
                         "sample": cpu_sample_text(w, args.workload, cores)},
        "e2e": {"value": val, "unit": w["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def dropin_e2e(steps: int = 30):
    """cfg2 frames/s as a C++ caller of the reference API sees them:
    svr::render / render_with_pools (raster.hpp) linked against
    libsvr_dropin.a + libsvr_b200.so (paper_2412_04459_b200/cpp/
    dropin_bench.cpp; host SparseScene in, five double Images out per call)."""
    exe = os.path.join(ROOT, "paper_2412_04459_b200", "cpp", "build", "dropin_bench")
    if not os.path.exists(exe):
        return {"value": None, "unit": "frames/s", "note": "dropin_bench not built"}
    try:
        r = subprocess.run([exe, str(steps)], capture_output=True, text=True, timeout=600)
        line = json.loads(r.stdout.strip().splitlines()[-1])
        d = line["dropin_fps"]
    except (subprocess.SubprocessError, ValueError, IndexError, KeyError) as e:
        return {"value": None, "unit": "frames/s", "note": f"dropin_bench failed: {e}"}
    return {"value": d["stats"], "unit": "frames/s", "train_pattern": d["train"],
            "cold_pattern": d["cold"], "steps": steps, "heap_tuned": line.get("heap_tuned"),
            "note": "svr::render through libsvr_dropin.a, wall clock per call, host SparseScene "
                    "in and five double Images out: value = unchanged scene (cache hit: content "
                    "fingerprints of the 250 MB scene + float->double images), train_pattern = "
                    "the caller's make_pools (400 MB of doubles) + render_with_pools after a "
                    "parameter change, cold_pattern = new geometry every call (full upload + "
                    "Morton tables); the caller keeps large blocks in its heap (mallopt)"}


# ------------------------------------------------------------------ ours
class RenderStep:
    """cfg2/cfg4 step: one view rendered into a resident frame."""

    def __init__(self, svr, ctx, scene, w, rank, world):
        self.svr, self.scene, self.w, self.rank, self.world = svr, scene, w, rank, world
        self.frame = svr.Frame(ctx)
        self.opts = svr.RenderOptions(K=1, supersample=1.0)
        self.cams = {}

    def cam(self, v):
        if v not in self.cams:
            self.cams[v] = make_camera(self.svr.ring_camera, self.w, v)
        return self.cams[v]

    def __call__(self, i):
        for v in view_ids(self.w, self.rank, self.world, i):
            self.svr.render_into(self.frame, self.scene, self.cam(v), self.opts)


class TrainStep:
    """cfg3/cfg5 step: ShardedTrainer over this rank's batch of views."""

    def __init__(self, svr, ctx, scene, w, rank, world):
        import torch
        from paper_2412_04459_b200.multiview import ShardedTrainer
        self.w, self.rank, self.world = w, rank, world
        self.views = sorted({v for i in range(4) for v in view_ids(w, rank, world, i)})
        dev = torch.device("cuda", ctx.device)
        cams, gts = {}, {}
        for v in self.views:
            cams[v] = make_camera(svr.ring_camera, w, v)
            gts[v] = torch.tensor(make_gt(w, v), device=dev)
        # ShardedTrainer indexes cameras/gts by view id
        idx = {v: k for k, v in enumerate(self.views)}
        self.idx = idx
        comm = None
        if world > 1 and os.environ.get("SVR_BENCH_BACKEND", "nccl") == "nccl":
            # the library's own NCCL communicator: the whole step (views, loss,
            # bucketed all-reduce of the flat registered buffer) is one
            # svr_train_batch_l1 call; the id travels over torch.distributed
            import torch.distributed as dist
            from paper_2412_04459_b200.multiview import NcclComm
            box = [NcclComm.make_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            comm = NcclComm(ctx, box[0], rank, world)
        self.trainer = ShardedTrainer(ctx, scene, [cams[v] for v in self.views],
                                      [gts[v] for v in self.views],
                                      svr.RenderOptions(K=1, supersample=1.0, training=True),
                                      comm=comm)
        self.loss = None

    def ids(self, i):
        return [self.idx[v] for v in view_ids(self.w, self.rank, self.world, i) if v in self.idx]

    def __call__(self, i):
        # the step's loss stays on the device (a one-element tensor): the
        # device-timed loop does not stall the host on a read-back between
        # steps, so the next step is enqueued while this one runs; the e2e
        # loop below reads every step's loss back to pinned host memory.
        # SVR_BENCH_SYNC_LOSS=1 reads it back inside each step instead.
        self.loss = self.trainer.step(self.ids(i), lazy=os.environ.get("SVR_BENCH_SYNC_LOSS") != "1")


class IterStep:
    """cfg3i step: one device training iteration (trainer.DeviceTrainer)."""

    def __init__(self, svr, ctx, scene, w, rank, world):
        import torch
        from paper_2412_04459_b200.trainer import DeviceTrainer
        self.cam = make_camera(svr.ring_camera, w, 0)
        self.gt_host = torch.tensor(make_gt(w, 0), dtype=torch.float32).pin_memory()
        self.gt = self.gt_host.to(torch.device("cuda", ctx.device))
        self.trainer = DeviceTrainer(svr, ctx, scene, svr.RenderOptions(K=1, supersample=1.0))
        self.frame = self.trainer.frame
        self.log = None

    def __call__(self, i):
        self.log = self.trainer.step(self.cam, self.gt)


def run_ours(args, rank, world, local_rank):
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2412_04459_b200 as svr

    w = WORKLOADS[args.workload]
    # one GPU per rank; SVR_BENCH_DEVICE / SVR_BENCH_BACKEND=gloo exist only to
    # exercise the multi-rank logic on a single-GPU box (tools/multirank_check.sh)
    dev = int(os.environ.get("SVR_BENCH_DEVICE", local_rank))
    backend = os.environ.get("SVR_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    local_rank = dev
    ctx = svr.Context(local_rank)
    arrays = make_scene_arrays(svr, w)
    scene = svr.Scene(ctx, arrays)
    step = {"render": RenderStep, "train": TrainStep, "iter": IterStep}[w["kind"]](
        svr, ctx, scene, w, rank, world)
    st = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local_rank))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    for i in range(max(3, args.warmup)):
        step(i)
    ctx.synchronize()
    torch.cuda.synchronize()
    if w["kind"] == "render":
        # Serving mode (svr_ctx_set_async): frames are enqueued whole, the
        # entry count is read back only when a result is consumed. One untimed
        # pass over the timed views sizes every frame's entry capacity; the
        # device counts any deferred frame that still outgrew it (reported).
        ctx.set_async(True)
        for i in range(args.steps):
            step(i)
            step.frame.info()
    ovf0 = ctx.overflow_count()
    if world > 1:
        dist.barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.15)
    ctx.enable_timing(True)
    ctx.stage_times(reset=True)
    launches0 = svr.launch_count()
    stats = []
    frame = step.trainer.frame if w["kind"] == "train" else step.frame
    for i in range(args.steps):
        with torch.cuda.stream(st):
            flush.zero_()
        ev[i][0].record(st)
        step(i)
        ev[i][1].record(st)
    ctx.synchronize()
    torch.cuda.synchronize()
    overflows = ctx.overflow_count() - ovf0
    inf = frame.info()  # the last timed step's frame
    stats.append((inf.n_entries, inf.n_visible, inf.sort_passes, inf.n_contribs))
    launches = svr.launch_count() - launches0
    stage = ctx.stage_times(reset=True)
    ctx.enable_timing(False)
    clk = clocks.stop()
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms_max = float(t.item())
    units_per_step = w["batch"]
    value = world * units_per_step * args.steps / (dev_ms_max / 1e3)

    # ---- e2e through the C ABI with host buffers ------------------------
    H = W = w["res"]
    lib = svr.load_library()
    if w["kind"] == "render":
        # Serving loop: three frames and three sets of pinned host images
        # rotate, so frame i's read-back (copy stream) overlaps the rendering
        # of the frames after it; every step still renders and reads back its
        # own five images (svr_frame_download_async / svr_frame_wait).
        # the five images, one copy each (SVR_BENCH_ONE_COPY=1: the frame's
        # contiguous SVR_BUF_OUTPUTS block in one copy; measured on one box
        # 1409 vs 1425 FPS for five copies, i.e. no gain: e2e sits at ~95 %
        # of the PCIe D2H rate either way)
        names = ([("OUTPUTS", 9)] if os.environ.get("SVR_BENCH_ONE_COPY") == "1" else
                 [("COLOR", 3), ("DEPTH", 1), ("MEDIAN_DEPTH", 1), ("NORMAL", 3), ("TRANSMITTANCE", 1)])
        pinned = [{k: torch.empty(H * W * c, dtype=torch.float32, pin_memory=True) for k, c in names}
                  for _ in range(3)]
        frames = [step.frame, svr.Frame(ctx), svr.Frame(ctx)]

        def e2e_step(i):
            f, host = frames[i % 3], pinned[i % 3]
            f.wait()  # host buffers of step i-3 consumed before they are reused
            for v in view_ids(w, rank, world, i):
                svr.render_into(f, scene, step.cam(v), step.opts)
            for k, buf in host.items():
                f.download_async(k, buf)

        def e2e_drain():
            for f in frames:
                f.wait()

        d2h = sum(b.numel() * 4 for b in pinned[0].values())
        h2d = C.sizeof(svr.svr_camera) + C.sizeof(svr.svr_render_options)
        e2e_note = ("scene resident on device (uploaded once); per step camera in, "
                    "color+depth+median+normal+transmittance out to pinned host memory; "
                    "three frames rotate so a step's read-back overlaps the next renders")
    elif w["kind"] == "iter":
        def e2e_step(i):
            step.gt.copy_(step.gt_host, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            step(i)  # returns the five loss values to the host

        def e2e_drain():
            pass

        d2h = 5 * 8
        h2d = H * W * 12 + C.sizeof(svr.svr_camera)
        e2e_note = ("scene, gradients and Adam moments resident on device; per step the ground "
                    "truth (pinned host) and camera in, the five loss values out")
    else:
        host_gt = {v: torch.tensor(make_gt(w, v)).pin_memory() for v in step.views}
        tr = step.trainer

        # the loss of step i is copied to pinned host memory behind the step
        # and read on the host one step later, so the host enqueues step i+1
        # while step i runs (the serving loop's pipelining, for training)
        loss_host = [torch.empty(1, dtype=torch.float32, pin_memory=True) for _ in range(2)]
        loss_ev = [None, None]
        losses = []

        def e2e_step(i):
            ids = step.ids(i)
            with torch.cuda.stream(tr.stream):
                for k in ids:
                    tr.gts[k].copy_(host_gt[step.views[k]], non_blocking=True)
            lt = tr.step(ids, lazy=True)
            with torch.cuda.stream(tr.stream):
                loss_host[i % 2].copy_(lt, non_blocking=True)
                loss_ev[i % 2] = torch.cuda.Event()
                loss_ev[i % 2].record(tr.stream)
            if i > 0:  # the previous step's loss, read on the host
                loss_ev[(i - 1) % 2].synchronize()
                losses.append(float(loss_host[(i - 1) % 2].item()))

        def e2e_drain():
            for ev in loss_ev:
                if ev is not None:
                    ev.synchronize()

        d2h = 4
        h2d = units_per_step * (H * W * 12 + C.sizeof(svr.svr_camera))
        e2e_note = ("scene and gradient buffers resident on device; per step each view's ground "
                    "truth (pinned host) and camera in, the loss out to pinned host memory "
                    "(read on the host one step later, so step i+1 is enqueued while step i runs)")
    # every rotating frame sizes its buffers for every view of the timed loop
    for i in range(max(args.e2e_steps, 6, args.warmup)):
        e2e_step(i)
    e2e_drain()
    ctx.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(args.e2e_steps):
        e2e_step(i)
    e2e_drain()
    ctx.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = world * units_per_step * args.e2e_steps / float(te.item())

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel --------------------------------
    E, n_vis, npass, contribs = stats[0]
    sw = int(np.ceil(args.supersample * w["res"]))
    ntiles = ((sw + 15) // 16) ** 2
    launches_per_step = {k: v / (args.steps * units_per_step) for k, v in stage.items()}
    per_step = {k: v / args.steps for k, v in stage.items()}
    cand = ["preprocess", "sort", "composite", "duplicate", "scan", "backward", "epilogue"]
    dom = max(cand, key=lambda k: per_step.get(k, 0.0))
    dd = dict(n_vox=arrays.n_voxels, n_pool=arrays.n_pool, n_vis=n_vis, E=E, R=sw * sw,
              ntiles=ntiles, stride=arrays.sh_stride, npass=npass, contribs=contribs)
    byt = stage_bytes(dom, dd)
    peak, peak_src = measured_peak_hbm()
    kernel_ms = launches_per_step[dom]  # one launch per view
    achieved = byt / (kernel_ms * 1e-3) / 1e9
    # the same kernel against the instruction-issue roof (4 schedulers x 148
    # SMs x max SM clock, one warp instruction each per cycle), from the
    # committed ncu instruction count of that kernel on this workload
    winst = traffic_from_profiles(dom + "_warp_inst", args.workload)
    issue_peak = 4 * 148 * 1e6 * float(clk.get("sm_mhz") or 1965.0)
    issue = None
    if winst:
        issue = {"bound": "issue", "achieved_warp_inst_per_s": winst / (kernel_ms * 1e-3),
                 "peak_warp_inst_per_s": issue_peak,
                 "frac": winst / (kernel_ms * 1e-3) / issue_peak,
                 "warp_inst_per_launch": winst, "source": "profiles/ncu_traffic.json"}
    binds = "issue" if issue and issue["frac"] > achieved / peak else "hbm"
    roofline = {"bound": "hbm", "binds": binds, "kernel": dom, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "issue": issue,
                "traffic": traffic_from_profiles(dom, args.workload, npass),
                "algorithmic_bytes": byt, "kernel_ms": kernel_ms, "peak_source": peak_src}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            rscene = ref.RefScene.from_arrays(arrays)
            cores = 1 if w["kind"] == "iter" else host_cores()
            opts = svr.RenderOptions(K=1, supersample=1.0, training=w["kind"] != "render")
            secs = cpu_step_fn(ref, rscene, w, args.workload, opts, svr.ring_camera, cores)(0)
            cpu = {"value": w["batch"] / secs, "unit": w["unit"], "cores": cores,
                   "kind": "reference", "sample": cpu_sample_text(w, args.workload, cores)}
        except Exception as e:  # the reference library may be absent on a fresh box
            cpu = {"value": None, "unit": w["unit"], "cores": host_cores(), "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}

    dropin = None
    if world == 1 and w["kind"] == "render" and w["scene"] == "G" and not args.no_dropin:
        dropin = dropin_e2e()

    config = bench_config(w, arrays.n_voxels, args.supersample)
    run = {"pool": arrays.n_pool, "entries_per_view": int(E), "visible_voxels": int(n_vis),
           "sort_passes": npass,
           "frames": ("deferred entry count (svr_ctx_set_async), "
                      f"{overflows} timed frame(s) outgrew their capacity"
                      if w["kind"] == "render" else "synchronous"),
           "parallelism": (f"view-sharded over {world} GPU(s), no data-path collective"
                           if w["kind"] == "render" else
                           f"replicas only ({world} independent iteration(s))"
                           if w["kind"] == "iter" else
                           f"view-batch sharded over {world} GPU(s), one in-place all-reduce "
                           f"of the flat gradient per step"),
           "precision": "projection/tile binning fp64 (bit-exact), compositing fp32"}
    if w["kind"] != "render":
        run["contribs_per_view"] = int(contribs)
        run["views_per_gpu_step"] = units_per_step
    line = {
        "metric": w["metric"], "value": value, "unit": w["unit"], "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (random-init parameters)",
        "mrays_per_s": value * sw * sw / 1e6,
        "config": config,
        "run": run,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": w["unit"], "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "note": e2e_note},
        "dropin_e2e": dropin,
        "gpu_launches": launches,
        "stage_ms_per_step": per_step,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        run_reference(args, rank)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
