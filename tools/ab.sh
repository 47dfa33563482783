#!/bin/bash
# A/B of library variants on one GPU: tools/ab.sh name1 name2 ... (built by tools/variants.py)
for v in "$@"; do
  TFG_LIB=paper_2507_01631_b200/_variants/$v/libtilefield_gpu.so timeout 150 python bench.py --no-cpu --no-render --steps 30 > gpurun_out/ab_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
l = [x for x in open(f"gpurun_out/ab_{v}.log") if x.startswith("{")]
if not l:
    print(v, "FAILED"); sys.exit()
d = json.loads(l[-1])
k = d["kernels"]
print(f"{v:10s} ms/step {d['ms_per_step']:.3f} value {d['value']/1e6:.2f}M " + " ".join(f"{n}={k[n]['ms_per_step']:.3f}" for n in k))
PY
done
