"""Summarise an ncu report (read here, no GPU): per-kernel time, DRAM bytes, throughput,
occupancy, issue, instruction count and top stall reasons.
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_rNN_<tag>.md
"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"), ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"), ("smsp__inst_executed.sum", "warp_inst"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_%"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts")]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    lines = [f"# ncu summary of `{rep}`", "", "| kernel | " + " | ".join(k[1] for k in KEYS) + " | top stalls |",
             "|" + "---|" * (len(KEYS) + 2)]
    for d in data:
        vals = []
        for k, _ in KEYS:
            v = d[ix[k]] if k in ix else ""
            u = units[ix[k]] if k in ix else ""
            vals.append(f"{v} {u}".strip())
        st = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[ix[h]] or 0) for h in stall}
        tot = sum(st.values()) or 1.0
        top = ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:4])
        lines.append(f"| {d[ix['Kernel Name']]} | " + " | ".join(vals) + f" | {top} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
