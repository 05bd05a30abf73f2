"""Summarise an ncu --set full report (.ncu-rep) into markdown for profiles/.

    python tools/ncu_summary.py gpurun_out/r1_k1_flow.ncu-rep "title" [alg_bytes] > profiles/x.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe % (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe cycles % (active)"),
    ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "FP64 tensor (DMMA) ops % of peak"),
    ("TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "FP64 pipe cycles % (elapsed)"),
    ("smsp__inst_executed.sum", "instructions"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, title = sys.argv[1], sys.argv[2]
    alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
    hdr, units, data = raw(rep)
    print(f"# {title}\n")
    print(f"Source report: `{rep}` (ncu --set full --clock-control none; one launch).\n")
    for row in data:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "kernel"
        print(f"## {name}\n")
        print("| metric | value | unit |\n|---|---|---|")
        vals = {}
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                vals[k] = row[i]
                print(f"| {label} (`{k}`) | {row[i]} | {units[i]} |")
        if alg and "dram__bytes_read.sum" in vals:
            i_r, i_w = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            traffic = float(row[i_r]) * scale[units[i_r]] + float(row[i_w]) * scale[units[i_w]]
            print(f"\nDRAM traffic {traffic / 1e6:.1f} MB vs algorithmic {alg / 1e6:.1f} MB "
                  f"(ratio {traffic / alg:.3f}).")
        stall = [(h, row[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                 and not h.endswith("_not_issued") and row[i] not in ("", "0")]
        if stall:
            tot = sum(float(v) for _, v in stall)
            print("\nWarp-stall sampling (share of samples):\n")
            for h, v in sorted(stall, key=lambda x: -float(x[1]))[:8]:
                print(f"- {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100 * float(v) / tot:.1f}%")
        print()


if __name__ == "__main__":
    main()
