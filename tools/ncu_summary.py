"""Markdown summary of ncu reports (one section per captured launch):
duration, DRAM bytes, SM / DRAM / FP64 pipe / DMMA utilisation, issue
activity, occupancy and the warp-stall sampling breakdown.

    python tools/ncu_summary.py gpurun_out/r1_k3.ncu-rep [...] > profiles/x.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("duration", "gpu__time_duration.sum"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue slots busy % (active)", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe cycles % (active)", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe cycles % (elapsed)", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("FP64 tensor (DMMA) ops % of peak", "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed"),
    ("DFMA thread instructions", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum"),
    ("DMUL thread instructions", "sm__sass_thread_inst_executed_op_dmul_pred_on.sum"),
    ("DADD thread instructions", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum"),
    ("warp instructions", "smsp__inst_executed.sum"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("registers/thread", "launch__registers_per_thread"),
    ("dynamic smem/block", "launch__shared_mem_per_block_dynamic"),
    ("warps active % (occupancy)", "sm__warps_active.avg.pct_of_peak_sustained_active"),
]
STALL = "smsp__pcsamp_warps_issue_stalled_"


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = [f"Source report: `{path}` (ncu --set full --clock-control none).", ""]
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        out.append(f"## {d.get('Kernel Name', '?')}")
        out.append("")
        out.append("| metric | value | unit |")
        out.append("|---|---|---|")
        vals = {}
        for label, m in METRICS:
            if m in d and d[m] != "":
                out.append(f"| {label} (`{m}`) | {d[m]} | {u.get(m, '')} |")
                try:
                    vals[m] = float(d[m].replace(",", ""))
                except ValueError:
                    pass
        if all(k in vals for k in ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "gpu__time_duration.sum")):
            fl = 2 * vals["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"] + \
                vals.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0) + \
                vals.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0)
            scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3}.get(
                u.get("gpu__time_duration.sum", "ns"), 1e-9)
            t = vals["gpu__time_duration.sum"] * scale
            if fl > 0:
                out.append(f"| FP64 FLOP/s (2 DFMA + DMUL + DADD) / duration | {fl / t / 1e12:.2f} | TFLOP/s |")
        stalls = {}
        for k, v in d.items():
            if k.startswith(STALL) and not k.endswith("_not_issued"):
                try:
                    stalls[k[len(STALL):]] = float(v.replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values())
        if tot > 0:
            out.append("")
            out.append("Warp-stall sampling (share of samples):")
            out.append("")
            for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]:
                out.append(f"- {k}: {100 * v / tot:.1f}%")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(summarise(p))
