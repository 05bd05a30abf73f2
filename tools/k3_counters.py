"""Summarise an ncu --csv counter log of the K3/K4 kernels: per kernel
template, launches, time, FP64 flops (2*DFMA + DMUL + DADD, SASS thread
counters) and the FP64 pipe utilisation.  Usage: k3_counters.py log.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ix = {k: h.index(k) for k in h}
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h) or not r[0].isdigit():
            continue
        per.setdefault((r[0], r[ix["Kernel Name"]]), {})[r[ix["Metric Name"]]] = (
            float(r[ix["Metric Value"]].replace(",", "")), r[ix["Metric Unit"]])
    agg = collections.OrderedDict()
    for (i, name), d in per.items():
        t, unit = d["gpu__time_duration.sum"]
        t_s = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9, "ms": 1e-3}.get(unit, 1e-9)
        fl = 2 * d["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"][0] + \
            d["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"][0] + \
            d["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"][0]
        key = name.split("(")[0].replace("unnamed>::", "").replace("void ", "")
        a = agg.setdefault(key, dict(n=0, t=0.0, fl=0.0, pipe_t=0.0))
        a["n"] += 1
        a["t"] += t_s
        a["fl"] += fl
        a["pipe_t"] += t_s * d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"][0]
    print("| kernel | launches | total us | FP64 TFLOP/s | FP64 pipe % (elapsed, time-weighted) |")
    print("|---|---|---|---|---|")
    for k, a in agg.items():
        print(f"| {k} | {a['n']} | {a['t'] * 1e6:.1f} | {a['fl'] / a['t'] / 1e12:.2f} | {a['pipe_t'] / a['t']:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
