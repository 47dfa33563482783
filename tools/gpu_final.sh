#!/bin/bash
# Round-end evidence on one GPU: build, GPU tests, the default bench line, the
# reference arm, and the ncu profile round.  usage: tools/gpu_final.sh <tag>
TAG=${1:-r02x}
python -c "import sys; sys.path.insert(0,'.'); from paper_2507_01631_b200 import build as b; b.build(); b.build_examples()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/${TAG}_gputest.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
bash tools/profile_round.sh ${TAG} mlp_bwd_kernel hash_fwd_kernel mlp_fwd_kernel raygen_kernel write_kernel composite_kernel adam_kernel accept_solve_kernel > gpurun_out/${TAG}_prof.log 2>&1
echo done
