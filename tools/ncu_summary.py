"""Flatten the details page of an ncu report into {"Section: Metric [unit]": value} JSON
(the summaries committed under profiles/; measurement tool, not product).

    python tools/ncu_summary.py REPORT.ncu-rep [kernel-regex] [note] > summary.json
"""
import csv
import io
import json
import re
import subprocess
import sys


def main(rep, kregex=".*", note=""):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if not re.search(kregex, d["Kernel Name"]):
            continue
        if "kernel" not in res:
            res = {"note": note, "kernel": d["Kernel Name"], "grid": d.get("Grid Size"),
                   "block": d.get("Block Size")}
        elif res["kernel"] != d["Kernel Name"]:
            break  # first matching launch only
        unit = f" [{d['Metric Unit']}]" if d.get("Metric Unit") else ""
        res[f"{d['Section Name']}: {d['Metric Name']}{unit}"] = d["Metric Value"]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
