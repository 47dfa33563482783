#!/usr/bin/env python
"""Writes profiles/<tag>_roofline.md from a bench.py JSON line: every
roofline number of the line recomputed from its inputs (algorithmic work per
unit x units, the measured per-phase time, the peaks of MEASURED_PEAKS.json /
profiles/red_peak.json), next to the ncu launch list's share of the step.

usage: python tools/roofline_report.py <bench.log> <tag> [launches.csv]
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    log, tag = sys.argv[1], sys.argv[2]
    launches = sys.argv[3] if len(sys.argv) > 3 else None
    line = next(json.loads(l) for l in open(log) if l.startswith("{"))
    S = line["config"]["samples_per_step_per_gpu"]
    B = line["config"]["rays_per_gpu_per_step"]
    hbm, tf_burst, tf_sust, src = bench.peaks()
    red = bench.red_peak()
    out = [f"# Roofline of bench line {tag}", "",
           f"Workload: {line['config']['workload']}; {B} rays and {S} samples per step per GPU; "
           f"{line['value'] / 1e6:.2f} M rays/s, {line['ms_per_step']:.3f} ms/step.", "",
           f"Peaks ({src}): HBM {hbm} GB/s, bf16 {tf_burst} TFLOP/s burst / {tf_sust} sustained"
           + (f"; random-index red.global.add {red['GBps']} GB/s (profiles/red_peak.json)" if red else "") + ".", "",
           "| family | ms/step | work per step | achieved | peak | frac |", "|---|---|---|---|---|---|"]
    for ph, k in line["kernels"].items():
        if ph not in bench.KERNEL_UNITS:
            continue
        bound, ps, pr, unit = bench.KERNEL_UNITS[ph]
        work = 28 * 1752595 if ph == "adam" else ps * S + pr * B
        sec = k["ms_per_step"] / 1e3
        if bound == "tensor":
            ach, peak, u = work / sec / 1e12, tf_sust, "TFLOP/s"
            wdesc = f"{ps} flop x {S} samples = {work / 1e9:.1f} GFLOP"
        else:
            ach, peak, u = work / sec / 1e9, hbm, "GB/s"
            wdesc = ("28 B x 1,752,595 params" if ph == "adam" else f"{ps} B x {S} samples + {pr} B x {B} rays") + \
                f" = {work / 1e6:.1f} MB"
        out.append(f"| {ph} | {k['ms_per_step']:.4f} | {wdesc} | {ach:.1f} {u} | {peak} | {ach / peak:.3f} |")
        if ph == "field_bwd" and red:
            rb = bench.SCATTER_BYTES * S
            ra = rb / sec / 1e9
            out.append(f"| field_bwd (scatter) | {k['ms_per_step']:.4f} | {bench.SCATTER_BYTES} B red payload x {S} "
                       f"samples = {rb / 1e6:.0f} MB | {ra:.1f} GB/s | {red['GBps']} | {ra / red['GBps']:.3f} |")
            rl_ = bench.red_lanes()
            if rl_:
                n = rl_["lane_reds_per_sample"] * S
                out.append(f"| field_bwd (scatter requests) | {k['ms_per_step']:.4f} | {rl_['lane_reds_per_sample']:.2f} "
                           f"red requests x {S} samples = {n / 1e6:.0f} M (ncu, profiles/red_lanes.json) | "
                           f"{n / sec / 1e9:.1f} G/s | {red['lanes_per_s'] / 1e9:.1f} G/s | "
                           f"{n / sec / red['lanes_per_s']:.3f} |")
    rl = line["roofline"]
    out += ["", f"Headline `roofline` of the line: kernel {rl['kernel']}, achieved {rl['achieved']:.2f} "
                f"{rl['unit']}, peak {rl['peak']}, frac {rl['frac']:.4f}; traffic (ncu DRAM bytes per launch, "
                f"profiles/traffic.json) {rl.get('traffic')}."]
    if "limiter" in rl:
        lm = rl["limiter"]
        out.append(f"Limiter: {lm['resource']}: {lm['achieved']:.1f} {lm['unit']} of {lm['peak']} = {lm['frac']:.3f}.")
        if "frac_requests" in lm:
            out.append(f"In red requests (the unit every red width shares: f32, v2 and v4 all sustain "
                       f"{lm['peak_requests_per_s'] / 1e9:.1f} G lane-requests/s in profiles/red_peak.json): "
                       f"{lm['red_requests_per_sample']:.2f} per sample, {lm['achieved_requests_per_s'] / 1e9:.1f} G/s "
                       f"= {lm['frac_requests']:.3f} of the peak.")
    if launches and os.path.exists(launches):
        rows = list(csv.reader(io.StringIO("".join(l for l in open(launches) if l.startswith('"')))))
        hdr = rows[0]
        ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = {}
        for r in rows[1:]:
            name = r[ik].split("(")[0].split("<")[0].replace("void ", "").replace("tfg::", "")
            agg[name] = agg.get(name, 0.0) + float(r[iv].replace(",", ""))
        tot = sum(agg.values())
        out += ["", f"ncu launch list ({os.path.basename(launches)}, cold-cache, serialised): share of GPU time",
                "", "| kernel | share |", "|---|---|"]
        for n, v in sorted(agg.items(), key=lambda x: -x[1])[:12]:
            out.append(f"| {n} | {100 * v / tot:.1f}% |")
    path = os.path.join(ROOT, "profiles", f"{tag}_roofline.md")
    open(path, "w").write("\n".join(out) + "\n")
    print(path)


if __name__ == "__main__":
    main()
