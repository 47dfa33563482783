#!/bin/bash
# Round profile on ONE GPU (run under gpurun): plain bench, ncu launch list,
# then one --set full capture per hot kernel, after the plain run exited 0,
# with the per-source-line (SASS) page exported for reading off-box.
# usage: tools/profile_round.sh <tag> [kernel regex ...]
set -e
TAG=${1:-rXX}
shift || true
KERNELS=${@:-mlp_bwd_kernel hash_fwd_kernel mlp_fwd_kernel raygen_kernel write_kernel composite_kernel adam_kernel accept_solve_kernel}
CMD="python bench.py --steps 2 --warmup 3 --no-render --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
for k in $KERNELS; do
  SKIP=3; [ "$k" = accept_solve_kernel ] && SKIP=1
  ncu --set full --clock-control none --import-source on -k regex:$k -s $SKIP -c 1 \
      -o gpurun_out/${TAG}_$k $CMD > gpurun_out/${TAG}_ncu_$k.log 2>&1 || echo "capture $k failed"
  ncu -i gpurun_out/${TAG}_$k.ncu-rep --page source --csv --print-source sass \
      > gpurun_out/${TAG}_${k}_source.csv 2>/dev/null || echo "source page $k failed"
done
echo done
