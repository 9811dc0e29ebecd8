"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py full  <report.ncu-rep> <out.json>
    python tools/ncu_summary.py launches <launches.csv> <out.json>

`full` extracts duration, DRAM/L2 bytes, pipe utilisation, issue activity and
the warp-stall breakdown of the first profiled kernel, plus the top stalled
SASS instructions from the source page.  `launches` turns the
`--metrics gpu__time_duration.sum` launch list into per-kernel totals/shares.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

NCU = "ncu"


def _raw(rep: str) -> dict:
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


_BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def _num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def full(rep: str, out: str) -> None:
    raw = _raw(rep)
    pick = [
        "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__block_size", "launch__grid_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_inst_executed_op_shared_atom.sum", "smsp__sass_inst_executed_op_global_red.sum",
        "smsp__sass_inst_executed_op_global_atom.sum",
    ]
    d = {k: (raw[k][0] if k == "Kernel Name" else _num(raw[k][0])) for k in pick if k in raw}
    d["units"] = {k: raw[k][1] for k in pick if k in raw and raw[k][1]}
    stalls = {}
    for k, (v, _) in raw.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            x = _num(v)
            if x:
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = x
    d["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda t: -t[1]))
    if d.get("dram__bytes_read.sum") is not None:
        # in bytes, whatever unit ncu chose for the raw fields (Mbyte, Gbyte, ...)
        d["dram_bytes_per_launch"] = sum(
            (d.get(k) or 0) * _BYTES.get(d["units"].get(k, "byte"), 1.0)
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    src = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) > 2:
        hdr = rows[1]
        try:
            i_s = hdr.index("Warp Stall Sampling (All Samples)")
            i_src = hdr.index("Source")
            i_ex = hdr.index("Instructions Executed")
            data = [r for r in rows[2:] if len(r) > i_s and r[i_s].isdigit()]
            tot = sum(int(r[i_s]) for r in data) or 1
            top = sorted(data, key=lambda r: -int(r[i_s]))[:15]
            d["top_stalled_sass"] = [{"share": round(int(r[i_s]) / tot, 4), "executed": r[i_ex],
                                      "sass": r[i_src].strip()} for r in top]
        except ValueError:
            pass
    with open(out, "w") as fh:
        json.dump(d, fh, indent=1)
    print(json.dumps({k: d[k] for k in list(d)[:8]}, indent=1))


def launches(path: str, out: str) -> None:
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = _num(r["Metric Value"])
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
        e = per.setdefault(name, {"launches": 0, "total_us": 0.0})
        e["launches"] += 1
        e["total_us"] += v * scale
    tot = sum(e["total_us"] for e in per.values()) or 1.0
    for e in per.values():
        e["share"] = round(e["total_us"] / tot, 4)
    res = {"total_us": tot, "kernels": dict(sorted(per.items(), key=lambda t: -t[1]["total_us"]))}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1)[:2000])


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
