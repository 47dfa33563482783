set -x
python -c "import sys; sys.path.insert(0,'.'); from paper_2507_01631_b200 import build as b; b.build(); b.build_examples()" > gpurun_out/build_b.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/red_peak tools/red_peak.cu && ./tools/bin/red_peak > gpurun_out/red_peak.json 2> gpurun_out/red_peak.err
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/gputest_b.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_b.log 2>&1
