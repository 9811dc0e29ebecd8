"""Diagnostic: wall time of set_reference's host prep vs the native call, per pair, 3 reps."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1709_06948_b200 as vmi
from paper_1709_06948_b200.synth import drive_sequence

scans, wp = drive_sequence(24)
eng = vmi.MIEngine(grid=vmi.GridSpec(resolution=1.0), binning=vmi.BinningSpec(kind=vmi.FeatureKind.VARZ))
for rep in range(3):
    row = []
    for i in range(23):
        t0 = time.perf_counter()
        pts = np.ascontiguousarray(scans[i][:, :3], dtype=np.float64)
        t1 = time.perf_counter()
        eng.ctx.set_reference_points(pts)
        t2 = time.perf_counter()
        row.append(f"{1e3*(t1-t0):.1f}/{1e3*(t2-t1):.1f}")
    print(f"rep {rep}: " + " ".join(row))
