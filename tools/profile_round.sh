#!/bin/bash
# Round profile on ONE GPU (run under gpurun): plain bench, ncu launch list,
# then one --set full capture per hot kernel, after the plain run exited 0.
# usage: tools/profile_round.sh <tag>
set -e
TAG=${1:-rXX}
CMD="python bench.py --steps 2 --warmup 3 --no-render --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
for k in mlp_bwd_kernel hash_fwd_kernel mlp_fwd_kernel raygen_kernel write_kernel composite_kernel adam_kernel accept_solve_kernel; do
  SKIP=3; [ "$k" = accept_solve_kernel ] && SKIP=1
  ncu --set full --clock-control none --import-source on -k regex:$k -s $SKIP -c 1 \
      -o gpurun_out/${TAG}_$k $CMD > gpurun_out/${TAG}_ncu_$k.log 2>&1 || echo "capture $k failed"
done
echo done
