"""Where the end-to-end time of a bench config goes (run on the GPU box):

    python tools/e2e_probe.py --config c2

Times, per call on the config's full pose batch: the host pose -> matrix
conversion, MIEngine.evaluate (host poses in, host MI out), the same through
host matrices (vmi_eval), the device-only launch, and best()."""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import bench
    import paper_1709_06948_b200 as vmi
    from paper_1709_06948_b200 import _lib

    wl = bench.workload(args.config, 1, bench.POSES_PER_GPU)
    eng = vmi.MIEngine(grid=vmi.GridSpec(resolution=wl.res),
                       binning=vmi.BinningSpec(kind=vmi.FeatureKind.from_name(wl.kind)), device=0)
    eng.set_reference(wl.a[:, :3].astype(np.float64), fetch=False)
    eng.set_query(wl.b)
    poses = wl.poses
    P = poses.shape[0]
    mats_h = _lib.poses_to_mats(poses)
    mats = torch.from_numpy(mats_h).cuda()
    mi = torch.empty(P, dtype=torch.float64, device="cuda")
    st = torch.empty(P, dtype=torch.int32, device="cuda")
    eng.evaluate(poses)
    eng.ctx.eval(mats_h)
    rows = {k: [] for k in ("conv", "evaluate", "eval_mats", "device", "device_split", "best")}
    head = max(2048, P // 32)
    for _ in range(args.reps):
        t0 = time.perf_counter()
        _lib.poses_to_mats(poses)
        rows["conv"].append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mi_e, _ = eng.evaluate(poses)
        rows["evaluate"].append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        eng.best(poses, mi_e)
        rows["best"].append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        eng.ctx.eval(mats_h)
        rows["eval_mats"].append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.ctx.eval_device(mats.data_ptr(), P, mi.data_ptr(), st.data_ptr())
        torch.cuda.synchronize()
        rows["device"].append(time.perf_counter() - t0)
        t0 = time.perf_counter()  # the head / tail launches vmi_eval_poses makes
        eng.ctx.eval_device(mats.data_ptr(), head, mi.data_ptr(), st.data_ptr())
        eng.ctx.eval_device(mats[head:].data_ptr(), P - head, mi[head:].data_ptr(),
                            st[head:].data_ptr())
        torch.cuda.synchronize()
        rows["device_split"].append(time.perf_counter() - t0)
    for k, v in rows.items():
        print(f"{args.config} {k:10s} {np.median(v) * 1e3:8.3f} ms  (min {np.min(v) * 1e3:.3f})")


if __name__ == "__main__":
    main()
