"""Per-config kernel ceilings for bench.py's `roofline` object (run here, on the CPU box).

    python tools/make_ceilings.py

Reads the ncu `--set full` summaries listed in SOURCES (written by
tools/ncu_summary.py from one capture of that config's K1 launch) and writes
profiles/ceilings.json: per config, DRAM bytes per launch (the `traffic`
field), warp-instructions per pose (-> the issue ceiling) and the FP64-pipe
active fraction (-> the FP64 ceiling).  bench.py reports a config's entry
only when it exists; it never reuses another config's capture.
"""

from __future__ import annotations

import json
import os

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
# config -> (summary file, poses in the captured launch)
SOURCES = {
    "c1": ("profiles/r02_v12_c1_k_pose_fast_full.json", 6069),
    "c1v": ("profiles/r02_v12_c1v_k_pose_fast_full.json", 6069),
    "c2": ("profiles/r02_v12_c2_k_pose_fast_full.json", 65536),
    "c3": ("profiles/r02_v12_c3_k_pose_fast_full.json", 970299),
    "c4": ("profiles/r02_v12_c4_k_pose_fast_full.json", 65536),
}


_BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def entry(path: str, poses: int) -> dict:
    d = json.load(open(os.path.join(ROOT, path)))
    ms = d["gpu__time_duration.sum"]
    inst = d["smsp__inst_executed.sum"]
    fp64 = d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"] / 100.0
    e = {
        "source": path,
        "kernel": d["Kernel Name"].split("(")[0],
        "poses_per_launch": poses,
        "ncu_kernel_ms": ms,
        "dram_bytes_per_launch": int(round(sum(
            d[k] * _BYTES[d["units"][k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum")))),
        "warp_inst_per_pose": inst / poses,
        "fp64_pipe_active_frac": fp64,
        "issue_active_frac": d["smsp__issue_active.avg.pct_of_peak_sustained_active"] / 100.0,
    }
    dp = [d.get(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum") for op in ("dfma", "dadd", "dmul")]
    if all(x is not None for x in dp):
        e["fp64_thread_ops_per_pose"] = sum(dp) / poses
    return e


def main() -> None:
    out = {cfg: entry(p, n) for cfg, (p, n) in SOURCES.items() if os.path.exists(os.path.join(ROOT, p))}
    out["_note"] = ("issue ceiling = 148 SMs x 4 schedulers x SM clock / warp_inst_per_pose; FP64 "
                    "ceiling = poses_per_launch / (ncu_kernel_ms x fp64_pipe_active_frac), i.e. the "
                    "rate if the FP64 pipe were busy every cycle with today's FP64 work")
    with open(os.path.join(ROOT, "profiles", "ceilings.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
