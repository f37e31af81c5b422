"""Top stalled SASS instructions of one kernel with their dominant stall reasons:
    python tools/ncu_stalls.py REPORT KERNEL_REGEX [SKIP] [N]"""
import csv
import io
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 15
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kre}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith("0x")]
    tot_i = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "(Not Issued)" not in c]
    total = sum(float(r[tot_i] or 0) for r in data) or 1.0
    top = sorted(range(len(data)), key=lambda i: -float(data[i][tot_i] or 0))[:n]
    for i in sorted(top):
        r = data[i]
        reasons = sorted(((float(r[c] or 0), h[c][6:]) for c in cols), reverse=True)[:2]
        print(f"{i:5d} {100 * float(r[tot_i]) / total:5.1f}%  {r[src][:48]:48s} " +
              ", ".join(f"{name} {100 * v / total:.1f}%" for v, name in reasons if v > 0))


if __name__ == "__main__":
    main()
