"""Summarises ncu outputs into profiles/ (launch-list shares, per-kernel key
metrics, and profiles/traffic.json = measured DRAM bytes per launch of each
bench kernel family, read by bench.py's roofline 'traffic' field).

usage: python tools/summarize_profiles.py <launches.csv> <tag> <prof.ncu-rep> [more.ncu-rep ...]

With the backward's source page (<tag>_mlp_bwd_kernel_source.csv) and the
plain bench line (<tag>_plain.log) beside its capture, also writes
profiles/red_lanes.json: the scatter's dynamic red count per sample (bench.py's
limiter reads it).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAMILY = {
    "mlp_bwd_kernel": "field_bwd",
    "mlp_fwd_kernel": "field_fwd",
    "hash_fwd_kernel": "field_fwd",
    "raygen_kernel": "sampler",
    "raygen_kernel<0>": "sampler",
    "raygen_kernel<1>": "sampler",
    "raygen_kernel<0, 2>": "sampler",
    "raygen_kernel<0, 8>": "sampler",
    "raygen_kernel<1, 2>": "sampler",
    "enc_half_kernel": "field_fwd",
    "import_plan_kernel": "sampler",
    "import_scatter_kernel": "sampler",
    "loss_reduce_kernel": "composite",
    "write_kernel": "sampler",
    "tiles_kernel": "sampler",
    "scan_reduce_kernel": "sampler",
    "scan_sums_kernel": "sampler",
    "scan_apply_kernel": "sampler",
    "composite_kernel": "composite",
    "adam_kernel": "adam",
    "grad_check_kernel": "adam",
    "occupancy_kernel": "occupancy",
    "accept_memo_kernel": "accept",
    "accept_solve_kernel": "accept",
    "accept_scatter_kernel": "accept",
}
METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem",
]


def family(k):
    # templated kernels (raygen_kernel<0, 2>, hash_fwd_kernel<0>, ...) by base name
    return FAMILY.get(k) or FAMILY.get(k.split("<")[0])


def short(name):
    n = name.split("(")[0]
    n = n.split("::")[-1]
    return n[5:] if n.startswith("void ") else n


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        agg[short(r[ki])][0] += 1
        agg[short(r[ki])][1] += float(r[vi].replace(",", ""))
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = collections.defaultdict(list)
    for r in rows[2:]:
        k = short(r[h.index("Kernel Name")])
        d = {}
        for m in METRICS:
            if m in h:
                v = r[h.index(m)]
                u = units[h.index(m)]
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    continue
                if u == "Mbyte":
                    x *= 1e6
                elif u == "Kbyte":
                    x *= 1e3
                elif u == "Gbyte":
                    x *= 1e9
                elif u in ("msecond", "ms"):
                    x *= 1e-3
                elif u in ("usecond", "us"):
                    x *= 1e-6
                elif u in ("nsecond", "ns"):
                    x *= 1e-9
                d[m] = x
        res[k].append(d)
    return res


def stalls(rep, top=3):
    """Top warp-stall reasons (sampled, all instructions) of the kernel in `rep`."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r]
    if not hi:
        return ""
    h = rows[hi[0]]
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = collections.Counter()
    for r in rows[hi[0] + 1:]:
        for i in cols:
            try:
                tot[h[i][6:]] += float(r[i] or 0)
            except (ValueError, IndexError):
                pass
    n = sum(tot.values()) or 1.0
    return ", ".join(f"{k} {100 * v / n:.0f}%" for k, v in tot.most_common(top))


RED_WIDTH = {"F32x4": 16, "F32x2": 8, "F32": 4}


def red_lanes(src_csv, plain_log):
    """Dynamic global-red counts of the captured backward launch by width
    (predicated-on thread instructions of REDG.E.ADD.F32[x2|x4] on its ncu
    source page) per sample of the bench step it was taken from."""
    rows = list(csv.reader(open(src_csv)))
    hi = [i for i, r in enumerate(rows) if "Address" in r and "Source" in r][0]
    h = rows[hi]
    ci = h.index("Predicated-On Thread Instructions Executed")
    by = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= ci:
            continue
        op = r[1].strip().split(" ")[0]
        if op.startswith("REDG.E.ADD.F32"):
            w = op.split(".")[3]
            by[w] += int(float(r[ci] or 0))
    line = [l for l in open(plain_log) if l.startswith("{")][-1]
    samples = json.loads(line)["config"]["samples_per_step_per_gpu"]
    lanes = sum(by.values())
    return {"lane_reds_per_launch": lanes, "by_width": dict(by),
            "red_bytes_per_launch": sum(n * RED_WIDTH[w] for w, n in by.items()),
            "samples_per_launch": samples, "lane_reds_per_sample": lanes / samples,
            "source": f"ncu source page of one mlp_bwd_kernel launch ({os.path.basename(src_csv)}), "
                      f"samples from the same command's plain bench line"}


def main():
    lpath, tag, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    agg = launches(lpath)
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu summary {tag}", "", "Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`,",
             "`python bench.py --steps 2 --warmup 3 --no-render --no-cpu`, `tools/profile_round.sh`; cold-cache, serialised:",
             "compare shares, not absolute times).", "",
             "| kernel | family | launches | ms/launch | share |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {family(k) or '-'} | {n} | {t / 1e6 / n:.3f} | {100 * t / tot:.1f}% |")
    r = collections.defaultdict(list)
    st = {}
    for rep in reps:
        for k, v in raw(rep).items():
            r[k] += v
            st[k] = stalls(rep)
    lines += ["", "Full captures (`ncu --set full --clock-control none`), one launch each:", "",
              "| kernel | time ms | DRAM read MB | DRAM write MB | SM % | DRAM % | L2 % | L1 % | tensor % | warps % | issue % | regs | top stalls |",
              "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = collections.defaultdict(float)
    for k, ds in r.items():
        d = ds[0]
        g = lambda m: d.get(m, float("nan"))
        lines.append(f"| {k} | {g('gpu__time_duration.sum') * 1e3:.3f} | {g('dram__bytes_read.sum') / 1e6:.1f} | "
                     f"{g('dram__bytes_write.sum') / 1e6:.1f} | {g('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{g('lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{g('l1tex__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{g('launch__registers_per_thread'):.0f} | {st.get(k, '')} |")
        fam = family(k)
        if fam:
            traffic[fam] += g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
        json.dump({k: v for k, v in traffic.items()}, f, indent=1)
    for rep in reps:
        src = rep.replace(".ncu-rep", "_source.csv")
        plain = os.path.join(os.path.dirname(rep), f"{tag}_plain.log")
        if "mlp_bwd_kernel" in rep and os.path.exists(src) and os.path.exists(plain):
            rl = red_lanes(src, plain)
            with open(os.path.join(ROOT, "profiles", "red_lanes.json"), "w") as f:
                json.dump(rl, f, indent=1)
            print("red lanes:", rl)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
