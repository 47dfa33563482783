#!/usr/bin/env python
"""Top stalled SASS instructions of an ncu source page export
(ncu -i rep --page source --csv --print-source sass).

usage: python tools/stall_top.py <source.csv> [n]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    col = "Warp Stall Sampling (All Samples)"
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[ix[col]] or 0) for r in data if len(r) > ix[col])
    print(f"total samples {tot:.0f}")
    agg = {s: sum(float(r[ix[s]] or 0) for r in data if len(r) > ix[s]) for s in stalls}
    print("by reason:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    top = sorted((r for r in data if len(r) > ix[col]), key=lambda r: -float(r[ix[col]] or 0))[:n]
    for r in top:
        why = sorted(((float(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:2]
        print(f"{100 * float(r[ix[col]]) / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:60]:60s} {why[0][1]} {why[1][1]}")


if __name__ == "__main__":
    main()
