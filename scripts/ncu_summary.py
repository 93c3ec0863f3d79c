"""Summarise an ncu report (--set full) into a small JSON/markdown table for profiles/.
usage: python scripts/ncu_summary.py report.ncu-rep out_prefix"""
import csv, io, json, subprocess, sys, collections

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
           "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size"]


def main(rep, prefix):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in h:
                d[m] = r[h.index(m)] + (" " + units[h.index(m)] if units[h.index(m)] else "")
        for i, w in enumerate(h):   # tensor-pipe utilisation (tcgen05 kernels)
            if (("tensor" in w or "pipe_tc" in w or "tcgen05" in w or "_tmem" in w or "utcmma" in w.lower()) and "pct" in w
                    and r[i] and r[i].strip() not in ("0", "0.0")):
                d[w] = r[i] + (" " + units[i] if units[i] else "")
        stalls = []
        for i, w in enumerate(h):
            if w.startswith("smsp__average_warps_issue_stalled_") and w.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((w[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(r[i])))
                except ValueError:
                    pass
        stalls.sort(key=lambda t: -t[1])
        d["top_stalls_per_issue"] = stalls[:6]
        out.append(d)
    json.dump(out, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu summary of `{rep.split('/')[-1]}`\n\n")
        for d in out:
            f.write(f"## {d['kernel']}\n\n")
            for k, v in d.items():
                if k not in ("kernel", "top_stalls_per_issue"):
                    f.write(f"- {k}: {v}\n")
            f.write("- top stalls (warps per issue): " + ", ".join(f"{a} {b:.2f}" for a, b in d["top_stalls_per_issue"]) + "\n\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
