"""Benchmark: batched MI candidate-pose evaluation on B200 (C2 workload).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path over one batch: score every candidate pose
of the batch (fused K1 kernel + exact fix-ups of flagged poses) and select the
np.argmax pose (device argmax; under torchrun a 16-byte NCCL all-gather of the
per-rank winners).  Workload: HDL-64-shaped synthetic scan
pair, 120,000 float32 points each, 1 m voxels, VARZ feature, 32 bins, phi
included; 65,536 poses per GPU uniform in truth ± (3 m, 3 m, 0.3 m, 1.5°, 1.5°,
10°).  Poses are sharded contiguously across ranks (weak scaling).

Prints ONE JSON line (rank 0).  `value` is device-timed with inputs resident in
HBM; `e2e` goes through the public MIEngine.evaluate API with host poses in
and host MI out.  `--impl reference` times the reference algorithm's CPU port
(oracle/, OpenMP over all host cores) on bounded samples of the same batch.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import socket
from dataclasses import dataclass
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TRUTH = (1.5, 0.3, 0.0, 0.0, 0.0, 0.05)
POSES_PER_GPU = 65536
METRIC = "MI pose evaluations/sec"
UNIT = "pose-evals/s"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--poses", type=int, default=POSES_PER_GPU, help="poses per GPU per step")
    ap.add_argument("--threads", type=int, default=0, help="CTA size (0 = library default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--rot", action="store_true",
                    help="pose grids: rotation-major path (vmi_eval_rot_device; measured slower "
                         "on B200, see DESIGN)")
    ap.add_argument("--config", default="c2", choices=["c1", "c1v", "c2", "c3", "c4", "c5"],
                    help="SURVEY.md 8(d) workload (c2 = the headline; c1v = C1's unordered "
                         "scans with the VARZ feature)")
    ap.add_argument("--frames", type=int, default=1001,
                    help="c5: frames in the synthetic drive (1001 frames = the 1000-pair sequence)")
    ap.add_argument("--c5-mode", default="nm", choices=["grid", "nm"],
                    help="c5: align_batch (voxmi.align-identical Nelder-Mead for every pair, "
                         "lockstep multi-pair kernel), or a 4,096-pose grid search per pair")
    ap.add_argument("--parity-sample", type=int, default=2048,
                    help="poses of the batch (strided) re-scored by the CPU oracle for the "
                         "line's `parity` object (0 = skip)")
    ap.add_argument("--dist-selftest", action="store_true",
                    help="launch plumbing only (CPU, gloo): ranks exchange synthetic shard "
                         "winners and rank 0 prints the pick; no GPU work")
    ap.add_argument("--c5-workers", type=int, default=6,
                    help="c5: host threads, each with its own engine/stream, so one pair's "
                         "A-grid build and uploads overlap another pair's pose scoring")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int | None:
    """`bench.py --gpus N` outside torchrun: re-exec this command under
    torch.distributed.run with N local ranks (one per GPU) and return its exit
    code.  Under torchrun (WORLD_SIZE set) the world must equal --gpus."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return None
    if args.gpus <= 1:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def init_dist(world: int, local: int):
    """One process group per run: NCCL over the GPUs (VMI_DIST_BACKEND=gloo for
    functional checks on fewer GPUs / CPU).  Returns (dist | None, collective device)."""
    import torch
    backend = os.environ.get("VMI_DIST_BACKEND", "nccl")
    if world <= 1:
        return None, "cpu"
    import torch.distributed as dist
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return dist, f"cuda:{local}"
    dist.init_process_group(backend)
    return dist, "cpu"


def exchange_winner(dist, cdev, value: float, index: int):
    """Per-rank (mi, global index) -> np.argmax's pick over all ranks (the one
    data-path collective: 8 + 8 bytes per rank, index as int64)."""
    from paper_1709_06948_b200.shard import all_gather_winner
    return all_gather_winner(value, index, dist, cdev)


def max_over_ranks(dist, cdev, x: float) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, cdev, x: float) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def run_dist_selftest(args, world, rank, local):
    """CPU check of the N-rank launch: contiguous shards of a synthetic MI
    vector, one winner exchange, rank 0 prints the pick (tests/test_bench.py)."""
    from paper_1709_06948_b200.shard import local_winner, shard_bounds
    os.environ.setdefault("VMI_DIST_BACKEND", "gloo")
    dist, cdev = init_dist(world, local)
    mi = np.random.default_rng(3).uniform(0, 1, size=args.poses)
    lo, hi = shard_bounds(mi.size, world, rank)
    v, i = local_winner(mi[lo:hi], lo)
    best, idx = exchange_winner(dist, cdev, v, i) if dist else (v, i)
    if rank == 0:
        print(json.dumps({"dist_selftest": True, "n_gpus": world, "best": best, "index": idx,
                          "want_index": int(np.argmax(mi))}), flush=True)
    if dist:
        dist.destroy_process_group()


def host_info(cores: int) -> dict:
    """CPU model, core count, numpy and BLAS build of the host running a CPU
    baseline (BASELINE.md 2 / SURVEY 8(d))."""
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")),
                         model)
    except OSError:
        pass
    blas = None
    try:
        import threadpoolctl
        b = [x for x in threadpoolctl.threadpool_info() if x.get("user_api") == "blas"]
        if b:
            blas = f"{b[0].get('internal_api')} {b[0].get('version')} ({b[0].get('architecture')})"
    except Exception:
        pass
    return {"cpu_model": model, "host_cpus": os.cpu_count(), "threads_used": cores,
            "numpy": np.__version__, "blas": blas,
            "oracle_build": "gcc -O2 -ffp-contract=off -fopenmp (oracle/Makefile)"}


@dataclass
class Workload:
    name: str
    a: np.ndarray          # scan A points (N, 3|4)
    b: np.ndarray          # scan B points / KITTI records
    poses: np.ndarray      # global candidate list (P, 6)
    res: float
    kind: str              # "varz" | "count"
    scaling: str           # "weak": poses per GPU fixed; "strong": global list fixed
    desc: str


def workload(cfg: str, world: int, per_gpu: int) -> Workload:
    """SURVEY.md §8(d) configurations (C2 is the headline)."""
    from paper_1709_06948_b200.geometry import EulerPose
    from paper_1709_06948_b200.synth import (LidarSceneSpec, candidate_batch, grid_poses,
                                             hdl64_pair)
    if cfg in ("c1", "c1v"):
        s = np.load(os.path.join(ROOT, "tests", "golden", "c1_scans.npz"))
        t = np.array([1.0, 0.5, 0.0, 0.0, 0.0, 0.1])
        poses = grid_poses(t, {"tx": t[0] + np.arange(-8, 9) * 0.25,
                               "ty": t[1] + np.arange(-8, 9) * 0.25,
                               "rz": t[5] + np.radians(np.arange(-10, 11) * 0.5)})
        kind = "count" if cfg == "c1" else "varz"
        return Workload(cfg, s["a"], s["b"], poses, 0.5, kind, "strong",
                        f"C1{'' if cfg == 'c1' else ' (VARZ variant)'}: reference "
                        f"synth_scene_pair(seed=0, 20k points, unordered), 0.5 m {kind.upper()}, "
                        "17x17x21 = 6069-pose (tx, ty, yaw) grid around the truth")
    if cfg == "c4":
        spec = LidarSceneSpec(extent=100.0, n_boxes=120, box_height=(1.0, 10.0))
        a, b = hdl64_pair(spec, EulerPose(*TRUTH))
        poses = candidate_batch(EulerPose(*TRUTH), per_gpu * world, seed=2024)
        return Workload("c4", a, b, poses, 0.2, "varz", "weak",
                        "C4: HDL-64-shaped 120k-point scans in a 100 m scene, 0.2 m VARZ "
                        "(large grid: hash-partitioned multi-pass table)")
    a, b = hdl64_pair(LidarSceneSpec(), EulerPose(*TRUTH))
    if cfg == "c3":
        t = np.asarray(TRUTH)
        poses = grid_poses(t, {
            "tx": t[0] + np.arange(-16, 17) * 0.625, "ty": t[1] + np.arange(-16, 17) * 0.625,
            "tz": t[2] + np.array([-0.5, 0.0, 0.5]),
            "rx": t[3] + np.radians([-1.0, 0.0, 1.0]), "ry": t[4] + np.radians([-1.0, 0.0, 1.0]),
            "rz": t[5] + np.radians(np.arange(-16, 17) * 1.25)})
        return Workload("c3", a, b, poses, 1.0, "varz", "strong",
                        "C3: C2 scans, wide 6-DOF grid 33x33x3x3x3x33 = 970,299 poses, "
                        "sharded across GPUs")
    poses = candidate_batch(EulerPose(*TRUTH), per_gpu * world, seed=2024)
    return Workload("c2", a, b, poses, 1.0, "varz", "weak",
                    "C2: HDL-64-shaped synthetic scan pair (120000 float32 points each), "
                    "1 m voxels, VARZ, 32 bins, phi included; candidate poses uniform in "
                    "truth +/- (3 m, 3 m, 0.3 m, 1.5 deg, 1.5 deg, 10 deg)")


def config(args, world, wl: Workload, P: int):
    return {
        "workload": wl.desc,
        "config_id": wl.name,
        "points": int(wl.b.shape[0]),
        "voxel_m": wl.res,
        "feature": wl.kind,
        "bins": 32,
        "poses_per_gpu": int(P),
        "global_batch": int(wl.poses.shape[0]),
        "parallelism": f"dp{world} (contiguous pose shards, NCCL all-gather of per-rank argmax)",
        "l2": "flushed between timed steps (256 MiB write); scan B (1.9 MB) is re-read from "
              "L2 by every pose within a step by design",
    }


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def profiled_ceilings(cfg: str):
    """This config's ncu-derived figures (profiles/ceilings.json, written by
    tools/make_ceilings.py from that config's own capture), or None."""
    p = os.path.join(ROOT, "profiles", "ceilings.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(cfg)
    except Exception:
        return None


def ceilings(c, value: float, sm_mhz: float | None):
    """Issue and FP64 ceilings (pose-evals/s) from this config's capture."""
    if not c:
        return None, None
    clk = (sm_mhz or 1965.0) * 1e6
    issue_rate = 148 * 4 * clk  # warp-instructions/s: 4 schedulers per SM, 1 issue/clk
    ic = issue_rate / c["warp_inst_per_pose"]
    fc = c["poses_per_launch"] / (c["ncu_kernel_ms"] * 1e-3 * c["fp64_pipe_active_frac"])
    issue = {"ceiling": ic, "unit": UNIT, "frac": value / ic,
             "warp_inst_per_pose": c["warp_inst_per_pose"],
             "issue_rate": issue_rate, "source": c["source"]}
    fp64 = {"ceiling": fc, "unit": UNIT, "frac": value / fc,
            "fp64_pipe_active_frac": c["fp64_pipe_active_frac"], "source": c["source"],
            "note": "rate if the FP64 pipe (DFMA 62 lanes/clk/SM measured, "
                    "profiles/r01_microbench_b200.txt) were busy every cycle"}
    return issue, fp64


def cpu_port_baseline(wl: Workload, poses, threads: int, budget_s: float = 15.0):
    """The reference algorithm's CPU port (oracle/, test infrastructure) on a
    bounded sample of the same batch; returns (poses/s, n_poses, cores)."""
    import oracle
    fa = oracle.feature_map(wl.a[:, :3].astype(np.float64), (0, 0, 0), wl.res, wl.kind)
    pts = wl.b[:, :3].astype(np.float64)
    cores = threads if threads > 0 else oracle.max_threads()
    # calibrate on a few poses, then size the sample to ~budget_s
    stride = max(1, poses.shape[0] // 4096)
    sample = poses[::stride]
    t0 = time.perf_counter()
    oracle.mi_objective_batch(fa, pts, oracle.poses_to_mats(sample[:cores]), res=wl.res,
                              threads=cores)
    per = (time.perf_counter() - t0) / cores
    n = int(min(sample.shape[0], max(cores, budget_s / max(per, 1e-6) * cores)))
    mats = oracle.poses_to_mats(sample[:n])
    t0 = time.perf_counter()
    oracle.mi_objective_batch(fa, pts, mats, res=wl.res, threads=cores)
    dt = time.perf_counter() - t0
    return n / dt, n, cores


def run_reference(args, world, rank):
    if rank != 0:
        return
    wl = workload(args.config, 1, args.poses)
    poses = wl.poses
    import oracle
    cores = oracle.max_threads()
    fa = oracle.feature_map(wl.a[:, :3].astype(np.float64), (0, 0, 0), wl.res, wl.kind)
    pts = wl.b[:, :3].astype(np.float64)
    # each step: a bounded, strided sample of the batch (~1-2 s of all-core CPU work)
    t0 = time.perf_counter()
    oracle.mi_objective_batch(fa, pts, oracle.poses_to_mats(poses[:cores]), res=wl.res,
                              threads=cores)
    per_pose = (time.perf_counter() - t0) / cores
    n = max(cores, int(1.5 / max(per_pose, 1e-6)) // cores * cores)
    stride = max(1, poses.shape[0] // n)
    times = []
    for s in range(args.warmup + args.steps):
        sel = poses[(s % stride)::stride][:n]
        mats = oracle.poses_to_mats(sel)
        t0 = time.perf_counter()
        mi, st = oracle.mi_objective_batch(fa, pts, mats, res=wl.res, threads=cores)
        int(np.argmax(mi))
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    value = n * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config(args, 1, wl, args.poses),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{n} strided poses of the {wl.name.upper()} batch per step, "
                                   f"OpenMP over {cores} host threads (oracle/voxmi_oracle.c)",
                         "host": host_info(cores)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def l2_flush(buf):
    buf.fill_(1)


def parity_check(eng, wl: Workload, poses, mi_gpu, st_gpu, n: int, n_hist: int = 16):
    """The CPU oracle (test infrastructure) on a strided sample of this step's
    batch, against the GPU's MI / status from the timed run: statuses equal,
    max relative MI error, the sample's argmax identical; histograms bit-exact
    on the first ``n_hist`` sampled poses."""
    import oracle
    P = poses.shape[0]
    stride = max(1, P // n)
    sel = np.arange(0, P, stride)[:n]
    fa = oracle.feature_map(wl.a[:, :3].astype(np.float64), (0, 0, 0), wl.res, wl.kind)
    pts = wl.b[:, :3].astype(np.float64)
    mats = oracle.poses_to_mats(poses[sel])
    t0 = time.perf_counter()
    omi, ost = oracle.mi_objective_batch(fa, pts, mats, res=wl.res, threads=0)
    dt = time.perf_counter() - t0
    g_mi, g_st = mi_gpu[sel], st_gpu[sel] & 0xFF
    ok = ost == 0
    rel = np.abs(g_mi[ok] - omi[ok]) / np.maximum(np.abs(omi[ok]), 1e-300)
    # np.argmax over the sample, GPU side with the library's near-tie re-score
    k_gpu, _ = eng.best(poses[sel], g_mi)
    _, h_st, hist, _ = eng.evaluate(poses[sel[:n_hist]], histograms=True)
    hist_ok = True
    for j in range(min(n_hist, sel.size)):
        _, s_o, c_o, _ = oracle.mi_objective_full(fa, pts, mats[j], res=wl.res)
        hist_ok &= bool(s_o == h_st[j] and np.array_equal(c_o, hist[j]))
    return {"sample": int(sel.size), "stride": int(stride),
            "status_equal": bool(np.array_equal(g_st, ost)),
            "max_rel_mi_err": float(rel.max()) if rel.size else 0.0,
            "argmax_equal": bool(k_gpu == int(np.argmax(omi))),
            "hist_bit_exact": f"{min(n_hist, sel.size)} poses: {'yes' if hist_ok else 'NO'}",
            "oracle_s": round(dt, 2),
            "checker": "oracle/voxmi_oracle.c (pinned to reference golden vectors)"}


def run_ours(args, world, rank, local):
    import torch
    import paper_1709_06948_b200 as vmi
    from paper_1709_06948_b200 import _lib
    from paper_1709_06948_b200.shard import shard_bounds

    # one rank per GPU; VMI_DIST_BACKEND=gloo exercises the N>1 code path on a
    # box with fewer GPUs (functional check only: ranks then share devices)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist, cdev = init_dist(world, local)
    wl = workload(args.config, world, args.poses)
    a, b, poses_all = wl.a, wl.b, wl.poses
    lo, hi = shard_bounds(poses_all.shape[0], world, rank)
    poses = poses_all[lo:hi]
    P = poses.shape[0]
    eng = vmi.MIEngine(grid=vmi.GridSpec(resolution=wl.res),
                       binning=vmi.BinningSpec(kind=vmi.FeatureKind.from_name(wl.kind)),
                       device=local, threads=args.threads)
    eng.set_reference(a[:, :3].astype(np.float64), fetch=False)
    eng.set_query(b)
    ctx = eng.ctx

    # algorithmic bytes per pose: 16*N_B + |V_B in AABB_A| + 8;
    # |V_B in AABB_A| measured from histograms of a strided sample
    _, _, hist, _ = eng.evaluate(poses[:: max(1, P // 256)], histograms=True)
    vb = float(np.mean(hist[:, :, 1:].sum(axis=(1, 2))))
    pts3 = np.asarray(b[:, :3])
    f32_exact = bool(np.all(pts3.astype(np.float32).astype(np.float64) == pts3))
    rec_bytes = 16.0 if f32_exact else 24.0  # float4 KITTI record, else 3 x f64
    bytes_per_pose = rec_bytes * b.shape[0] + vb + 8.0

    stream = torch.cuda.Stream(device=local)
    mats_h = _lib.poses_to_mats(poses)
    mats = torch.from_numpy(mats_h).to(f"cuda:{local}")
    # pose grids (C1, C3): rotation-major -- scan B rotated once per distinct
    # rotation, the point loop reads the rotated copy (vmi_eval_rot_device);
    # the plan (grouping + permutation) is host preprocessing of the poses,
    # like poses_to_mats; the rotation kernel itself is inside the timed step
    rots_h, pm_h, ridx_h, perm_h = _lib.rotation_plan(poses, mats_h)
    use_rot = args.rot and rots_h.shape[0] * 16 <= P
    if use_rot:
        dv = f"cuda:{local}"
        d_rots, d_pm = torch.from_numpy(rots_h).to(dv), torch.from_numpy(pm_h).to(dv)
        d_ridx, d_perm = torch.from_numpy(ridx_h).to(dv), torch.from_numpy(perm_h).to(dv)
    mi = torch.empty(P, dtype=torch.float64, device=f"cuda:{local}")
    st = torch.empty(P, dtype=torch.int32, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    fixups_total = 0

    def step(ev=None):
        nonlocal fixups_total
        s = stream.cuda_stream
        if ev:
            ev[0].record(stream)
        if use_rot:  # rotate + point loop + fix-ups + scatter to pose order
            x0 = ctx.counters()["exact_poses"]
            ctx.eval_rot_device(d_rots.data_ptr(), rots_h.shape[0], d_pm.data_ptr(),
                                d_ridx.data_ptr(), d_perm.data_ptr(), P, mi.data_ptr(),
                                st.data_ptr(), stream=s)
            if ev:
                ev[1].record(stream)
            fixups_total += ctx.counters()["exact_poses"] - x0
        else:
            ctx.eval_device(mats.data_ptr(), P, mi.data_ptr(), st.data_ptr(), stream=s)
            if ev:
                ev[1].record(stream)
            fixups_total += ctx.eval_fixups(mats.data_ptr(), P, mi.data_ptr(), st.data_ptr(),
                                            stream=s)
        best, idx = ctx.argmax_device(mi.data_ptr(), P, stream=s)
        if dist is not None:
            with torch.cuda.stream(stream):
                return exchange_winner(dist, cdev, best, lo + idx)
        return best, lo + idx

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = ctx.launches
    fixups_total = 0
    step_ms, kern_ms = [], []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            l2_flush(flush)
            torch.cuda.synchronize()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[2].record(stream)  # step start (before the kernel-start event)
            step((e[0], e[1]))
            e_end = torch.cuda.Event(enable_timing=True)
            e_end.record(stream)
            e_end.synchronize()
            step_ms.append(e[2].elapsed_time(e_end))
            kern_ms.append(e[0].elapsed_time(e[1]))
    torch.cuda.synchronize()
    launches = ctx.launches - launches0
    total_ms = max_over_ranks(dist, cdev, float(sum(step_ms)))
    if dist:
        dist.barrier()
    n_total = poses_all.shape[0]  # all ranks' poses (shards cover the global list)
    value = n_total * args.steps / (total_ms / 1e3)
    mi_h = mi.cpu().numpy()
    st_h = st.cpu().numpy()

    # end to end through the public API: host poses in (pose->matrix on host,
    # H2D), host MI out (D2H), host argmax + near-tie re-score (best); max over ranks
    e2e_times = []
    eng.evaluate(poses)  # untimed: first call allocates the host-API staging buffers
    for _ in range(args.e2e_steps):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        mi_e, _ = eng.evaluate(poses)
        eng.best(poses, mi_e)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(dist, cdev, float(np.mean(e2e_times)))
    e2e_value = n_total / e2e_s

    kern_s = float(np.mean(kern_ms)) / 1e3
    achieved = bytes_per_pose * P / kern_s / 1e9
    peak, peak_src = measured_peak()
    clk = clocks.summary()
    prof = profiled_ceilings(wl.name)
    issue_c, fp64_c = ceilings(prof, P / kern_s, clk.get("sm_mhz"))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": wl.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(config(args, world, wl, P), rotation_major=(
            f"{rots_h.shape[0]} distinct rotations: scan B rotated once per rotation (k_rotate, "
            "inside the timed step), the point loop reads the rotated copy" if use_rot else False)),
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_src,
            "traffic": prof["dram_bytes_per_launch"] if prof else None,
            "traffic_source": (f"{prof['source']} ({prof['poses_per_launch']} poses per launch)"
                               if prof else "no ncu capture of this config"),
            "kernel": ("k_pose_fast (K1, fused transform/voxelize/aggregate/histogram/MI)"
                       + (" ROT instantiation (pre-rotated double4 records) + k_rotate + fix-up "
                          "check + scatter to pose order" if use_rot else "")),
            "kernel_ms": kern_s * 1e3,
            "algorithmic_bytes_per_pose": bytes_per_pose,
            "mean_vb_in_aabb_a": vb,
            "bytes_formula": f"{int(rec_bytes)}*N_B + |V_B in AABB_A| + 8",
            "issue_ceiling": issue_c,
            "fp64_ceiling": fp64_c,
        },
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": int(P * 96 + ((P * 12 + rots_h.shape[0] * 96)
                                                    if use_rot and P >= 4096 else 0)),
                "d2h_bytes_per_step": int(P * 12),
                "path": "MIEngine.evaluate(host poses P x 6 f64) -> host MI + status, "
                        "MIEngine.best (np.argmax + near-tie re-score); H2D = the P x 12 f64 "
                        "pose matrices built on the host (pinned staging), D2H = MI f64 + "
                        "status i32"},
        "gpu_launches": int(launches),
        "fixups_per_step": fixups_total / args.steps,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and args.parity_sample > 0:
        line["parity"] = parity_check(eng, wl, poses, mi_h, st_h, args.parity_sample)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, n, cores = cpu_port_baseline(wl, poses, threads=1)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"{n} strided poses of the {wl.name.upper()} batch, "
                                          "single thread (oracle/voxmi_oracle.c)",
                                "host": host_info(cores)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if dist:
        dist.destroy_process_group()


def run_c5(args, world, rank, local):
    """C5: consecutive scan pairs of a synthetic drive (1000 pairs at the
    default 1001 frames).  --c5-mode nm (default): every pair aligned exactly as
    voxmi.align does (Nelder-Mead from a prior perturbed by 0.5 m / 1 deg), all
    pairs of a rank's shard resident at once and advanced in lockstep
    (align_batch: one multi-pair kernel launch per step); --c5-mode grid: a
    4,096-pose (tx, ty, yaw) grid search per pair on host worker threads.  One
    step = every pair of the shard aligned, scan A grids built on the GPU
    included.  Wall-clock timed, max over ranks; pairs sharded contiguously."""
    import torch
    import paper_1709_06948_b200 as vmi
    from paper_1709_06948_b200.shard import shard_bounds
    from paper_1709_06948_b200.synth import C5_SIMPLEX_STEPS, c5_grid, c5_priors, drive_sequence
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist, cdev = init_dist(world, local)
    # each rank builds only the frames of its pair shard (frame generation is
    # host work outside the timed region; spawned processes, cores shared by ranks)
    n_frames = args.frames
    pairs = list(range(n_frames - 1))
    lo, hi = shard_bounds(len(pairs), world, rank)
    gen_workers = max(1, (os.cpu_count() or 1) // int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    scans, world_poses = drive_sequence(n_frames, workers=min(32, gen_workers), subset=(lo, hi + 1))
    priors, truths = c5_priors(world_poses)
    mine = list(range(lo, hi))
    cfg = vmi.AlignmentConfig(simplex=vmi.SimplexConfig(initial_steps=C5_SIMPLEX_STEPS))

    def terr(i, est):
        t = truths[i]
        return float(np.hypot(est[0] - t.tx, est[1] - t.ty))

    extra = {}
    if args.c5_mode == "nm":
        eng = vmi.MIEngine(grid=cfg.grid, binning=cfg.binning, include_phi=cfg.phi_enabled,
                           device=local)
        # the drive's scans as a KITTI loader leaves them: float32 records in
        # page-locked memory (scan_io.load_kitti_bin(pinned=True)); their
        # upload to the GPU is inside every timed step
        from paper_1709_06948_b200.scan_io import pinned_copy
        pin = {i: pinned_copy(scans[i]) for i in range(lo, hi + 1)}
        my_pairs = [(pin[i], pin[i + 1]) for i in mine]
        t0s = [vmi.euler_to_transform(vmi.EulerPose.from_vector(priors[i])) for i in mine]
        for _ in range(max(1, args.warmup)):  # (sizes the engine's grow-only buffers)
            vmi.align_batch(my_pairs, t0s, cfg, engine=eng)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        stats = {}
        acc = {}
        launches0 = eng.ctx.launches
        t0 = time.perf_counter()
        for _ in range(args.steps):
            reps = vmi.align_batch(my_pairs, t0s, cfg, engine=eng, stats=stats)
            for k in ("set_pairs_s", "wall_time", "final_eval_s", "reports_s"):
                acc[k] = acc.get(k, 0.0) + stats[k] / args.steps
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        launches = eng.ctx.launches - launches0
        cnt = eng.ctx.counters()
        errs = [terr(i, r.estimated_pose.as_vector()) for i, r in zip(mine, reps)]
        n_evals = sum_over_ranks(dist, cdev, float(stats["evaluations"]) * args.steps)
        extra = {"redone_exact": int(sum_over_ranks(dist, cdev, float(stats["redone_exact"]))),
                 "gpu_launches_per_step": launches / args.steps,
                 "nm_wall_s_per_step": stats["wall_time"],
                 "breakdown_s_per_step": {k: round(v, 4) for k, v in acc.items()},
                 "nm_steps_per_step": cnt["nm_steps"] / (args.steps + max(1, args.warmup)),
                 "nm_probes_per_step": cnt["nm_probes"] / (args.steps + max(1, args.warmup)),
                 "input": "float32 KITTI records in pinned host memory, uploaded every step"}
        eng.close()
    else:
        from concurrent.futures import ThreadPoolExecutor
        nw = max(1, args.c5_workers)
        engines = [vmi.MIEngine(grid=cfg.grid, binning=cfg.binning, device=local)
                   for _ in range(nw)]

        def align_pair(eng, i):
            eng.set_reference(scans[i][:, :3], fetch=False)
            eng.set_query(scans[i + 1])
            poses = c5_grid(priors[i])
            mi, _ = eng.evaluate(poses)
            k, _ = eng.best(poses, mi)
            return poses[k]

        def worker(w):
            return [terr(i, align_pair(engines[w], i)) for i in mine[w::nw]]

        with ThreadPoolExecutor(nw) as pool:
            for _ in range(max(1, args.warmup)):
                list(pool.map(lambda w: [align_pair(engines[w], i) for i in mine[w::nw][:1]],
                              range(nw)))
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            errs = []
            t0 = time.perf_counter()
            for _ in range(args.steps):
                errs = [e for r in pool.map(worker, range(nw)) for e in r]
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        n_evals = sum_over_ranks(dist, cdev, float((hi - lo) * args.steps * 4096))
        extra = {"host_workers": nw}
        for e in engines:
            e.close()
    # every rank's wall time (max) and pair count (sum): the job's alignments/s
    dt = max_over_ranks(dist, cdev, dt)
    n = int(sum_over_ranks(dist, cdev, float((hi - lo) * args.steps)))
    if rank == 0:
        line = {
            "metric": "scan-pair alignments/sec", "value": n / dt, "unit": "alignments/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5: {n_frames}-frame synthetic drive (HDL-64-shaped "
                                   "120k-point scans ~1 m apart), consecutive pairs, 1 m VARZ; per "
                                   "pair: GPU A-grid build + "
                                   + ("voxmi.align-identical Nelder-Mead from a prior perturbed by "
                                      "0.5 m / 1 deg (lockstep over all pairs)"
                                      if args.c5_mode == "nm" else
                                      "16x16x16 (tx, ty, yaw) grid around the prior"),
                       "pairs": len(pairs), "mode": args.c5_mode, "timing": "wall clock"},
            "pose_evals_per_s": n_evals / dt,
            "median_translation_error_m": float(np.median(errs)) if errs else None,
            **extra,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_reference_c5(args, world, rank):
    """C5 reference arm: the reference's serial align loop (oracle/nm.py on the
    oracle's mi_objective, CPU port) on a bounded number of the drive's pairs,
    one pair per host thread (all cores)."""
    if rank != 0:
        return
    import oracle
    from oracle.nm import align_pair
    from concurrent.futures import ThreadPoolExecutor
    from paper_1709_06948_b200.synth import C5_SIMPLEX_STEPS, c5_priors, drive_sequence
    cores = oracle.max_threads()
    n = max(1, min(cores, args.frames - 1))
    scans, wp = drive_sequence(args.frames, workers=min(32, cores), subset=(0, n + 1))
    priors, truths = c5_priors(wp)
    with ThreadPoolExecutor(cores) as pool:
        times = []
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = list(pool.map(lambda i: align_pair(scans[i][:, :3], scans[i + 1][:, :3],
                                                     priors[i], C5_SIMPLEX_STEPS), range(n)))
            if s >= args.warmup:
                times.append(time.perf_counter() - t0)
    value = n * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": "scan-pair alignments/sec", "value": value,
        "unit": "alignments/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C5: the first {n} pairs of the {args.frames}-frame drive, "
                               "voxmi.align's serial Nelder-Mead per pair", "mode": "nm"},
        "cpu_baseline": {"value": value, "unit": "alignments/s", "cores": cores, "kind": "port",
                         "sample": f"{n} pairs per step, one pair per host thread "
                                   "(oracle/nm.py on oracle/voxmi_oracle.c)",
                         "host": host_info(cores)},
        "e2e": {"value": value, "unit": "alignments/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "median_iterations": float(np.median([r[2] for r in res])),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rc = self_launch(args)
    if rc is not None:  # --gpus N outside torchrun: the ranks ran as children
        sys.exit(rc)
    world, rank, local = dist_env()
    if args.dist_selftest:
        run_dist_selftest(args, world, rank, local)
    elif args.config == "c5" and args.impl != "reference":
        run_c5(args, world, rank, local)
    elif args.config == "c5":
        run_reference_c5(args, world, rank)
    elif args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
