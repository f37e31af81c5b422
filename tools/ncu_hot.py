"""Top stalled SASS instructions of one kernel in an ncu report (needs -lineinfo builds):
    python tools/ncu_hot.py REPORT KERNEL_BASE_REGEX [SKIP] [N]   (SKIP-th matching launch)"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{kre}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(rows[0][1] if rows and len(rows[0]) > 1 else "?")
    his = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    hi = his[0]
    h = rows[hi]
    end = his[1] if len(his) > 1 else len(rows)
    data = [r for r in rows[hi + 1:end] if len(r) == len(h) and r[0].startswith("0x")]
    si = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")
    tot = sum(int(r[si]) for r in data) or 1
    print(f"samples {tot}, instructions {len(data)}")
    top = sorted(range(len(data)), key=lambda i: -int(data[i][si]))[:n]
    for i in sorted(top):
        r = data[i]
        print(f"{i:5d} {100 * int(r[si]) / tot:5.1f}%  {r[src].strip()[:110]}")
    c = Counter()
    for r in data:
        ins = r[src].strip().split()
        if not ins:
            continue
        op = ins[1] if ins[0].startswith("@") and len(ins) > 1 else ins[0]
        c[op.split(".")[0]] += int(r[si])
    print("by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in c.most_common(14)))


if __name__ == "__main__":
    main()
