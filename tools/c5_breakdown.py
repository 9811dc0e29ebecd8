"""Per-stage wall-clock breakdown of C5 alignments (diagnostic).

usage: python tools/c5_breakdown.py [frames]
"""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1709_06948_b200 as vmi
from paper_1709_06948_b200.synth import drive_sequence, grid_poses, relative_pose

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 6
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if os.environ.get("NOGC"):
    import gc
    gc.disable()
scans, wp = drive_sequence(frames)
eng = vmi.MIEngine(grid=vmi.GridSpec(resolution=1.0), binning=vmi.BinningSpec(kind=vmi.FeatureKind.VARZ))
offs = np.linspace(-0.75, 0.75, 16); yo = np.radians(np.linspace(-1.5, 1.5, 16))
for rep in range(reps):
    tot = 0.0
    for i in range(frames - 1):
        t = relative_pose(wp[i], wp[i + 1]); c = np.array([t.tx, t.ty, 0, 0, 0, t.rz])
        torch.cuda.synchronize(); t0 = time.perf_counter()
        eng.set_reference(scans[i][:, :3], fetch=False); t1 = time.perf_counter()
        eng.set_query(scans[i + 1]); t2 = time.perf_counter()
        poses = grid_poses(c, {"tx": c[0] + offs, "ty": c[1] + offs, "rz": c[5] + yo}); t3 = time.perf_counter()
        mi, st = eng.evaluate(poses); t4 = time.perf_counter()
        k, b = eng.best(poses, mi); t5 = time.perf_counter()
        tot += t5 - t0
        if rep and (t5 - t0) > 0.012:
            print(f"pair {i:2d} pts {len(scans[i])}/{len(scans[i + 1])} ref {1e3*(t1-t0):6.2f} ms  "
                  f"query {1e3*(t2-t1):6.2f}  grid {1e3*(t3-t2):5.2f}  eval {1e3*(t4-t3):6.2f}  "
                  f"best {1e3*(t5-t4):5.2f}")
    print(f"rep {rep}: {frames - 1} pairs in {1e3 * tot:.1f} ms -> {(frames - 1) / tot:.1f} pairs/s")
