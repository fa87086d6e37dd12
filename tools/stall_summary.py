"""Aggregate warp-stall samples from an `ncu --page source --csv` export.

usage: python tools/stall_summary.py gpurun_out/source_<w>.csv [--top N]
Prints total samples per stall reason, and the instructions with most samples.
"""
import csv
import sys
from collections import Counter


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 15
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = Counter()
    per = []
    for r in body:
        s = 0
        for i in stall_cols:
            v = int(r[i] or 0)
            tot[hdr[i]] += v
            s += v
        per.append((s, r[1].strip(), {hdr[i]: int(r[i] or 0) for i in stall_cols if int(r[i] or 0)}))
    allv = sum(tot.values())
    print(f"{path}: {allv} samples, {len(body)} instructions")
    for k, v in tot.most_common():
        if v:
            print(f"  {k:28s} {v:9d} {v / allv:6.1%}")
    print("top instructions:")
    for s, src, d in sorted(per, key=lambda x: -x[0])[:top]:
        dd = ", ".join(f"{k[6:]}={v}" for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:4])
        print(f"  {s:8d} {src[:60]:60s} {dd}")


if __name__ == "__main__":
    main()
