"""Time K1 at C4 for several table pass counts (planner tuning; GPU only).

    python tools/pass_sweep.py [npass ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1709_06948_b200 as vmi  # noqa: E402

wl = bench.workload("c4", 1, 16384)
eng = vmi.MIEngine(grid=vmi.GridSpec(resolution=wl.res),
                   binning=vmi.BinningSpec(kind=vmi.FeatureKind.VARZ), device=0)
eng.set_reference(wl.a[:, :3].astype(np.float64))
eng.set_query(wl.b)
dev = torch.device("cuda", 0)
mats = torch.from_numpy(eng.mats(wl.poses)).to(dev)
P = mats.shape[0]
mi = torch.empty(P, dtype=torch.float64, device=dev)
st = torch.empty(P, dtype=torch.int32, device=dev)
s = torch.cuda.current_stream(dev).cuda_stream
for npass in [int(x) for x in sys.argv[1:]] or [0, 2, 3, 4, 5, 6, 8]:
    eng.ctx.set_passes(npass)
    for _ in range(2):
        eng.ctx.eval_device(mats.data_ptr(), P, mi.data_ptr(), st.data_ptr(), stream=s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        eng.ctx.eval_device(mats.data_ptr(), P, mi.data_ptr(), st.data_ptr(), stream=s)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    flagged = int(((st.cpu().numpy() & 0x100) != 0).sum())
    print(f"npass {npass}: {ms / 3:.2f} ms / {P} poses, flagged {flagged}", flush=True)
