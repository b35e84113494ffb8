"""Per-kernel totals and shares of an ncu launch list (--metrics gpu__time_duration.sum
--csv --log-file ...; measurement tool). Times are ncu's serialised cold-cache
per-launch durations: compare SHARES with the CUDA-event stage times, not absolutes.

    python tools/launch_summary.py launches.csv [note] > summary.json
"""
import csv
import json
import sys
from collections import defaultdict


def main(path, note=""):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0]
        tot[name] += float(r[iv].replace(",", ""))
        cnt[name] += 1
    all_ns = sum(tot.values())
    out = {"note": note, "launches": sum(cnt.values()), "total_ms": all_ns / 1e6,
           "kernels": [{"name": k, "launches": cnt[k], "ms": tot[k] / 1e6,
                        "share": tot[k] / all_ns}
                       for k in sorted(tot, key=lambda k: -tot[k])]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
