"""Per-stage DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum, bytes per launch) of one
ITA iteration from an `ncu --set full` report holding one launch of each sweep (matched by kernel
name: az_cluster_kernel<L, 2 | 5 | 6>, rg_sweep_kernel<L, 1 | 0, 0, 0>); writes the JSON bench.py
reads for the roofline 'traffic' field.
    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep profiles/traffic_c3.json"""
import csv
import io
import json
import re
import subprocess
import sys

STAGES = ["S1_az_head", "S2_rg_G", "S3_az_resid", "S4_rg_M", "S5_az_tail"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    res = {"source": rep, "kernels": {}}
    pat = {"S1_az_head": r"az_cluster_kernel<\d+, 2>", "S2_rg_G": r"rg_sweep_kernel<\d+, 1, 0, 0>",
           "S3_az_resid": r"az_cluster_kernel<\d+, 5>", "S4_rg_M": r"rg_sweep_kernel<\d+, 0, 0, 0>",
           "S5_az_tail": r"az_cluster_kernel<\d+, 6>"}
    for stage in STAGES:
        d = next(r for r in data if re.search(pat[stage], r[ix["Kernel Name"]]))
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[ix[k]]) * SCALE[units[ix[k]]]
        res[stage] = b
        res["kernels"][stage] = d[ix["Kernel Name"]]
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
