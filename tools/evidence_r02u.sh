#!/bin/bash
# Reproducible replacements for round-1 scratch measurements cited in DESIGN.md §6 / §9c:
# FP64 pipe latency / throughput, strip-height variants of the two-sweep pass (solve time),
# per-kernel times incl. one RAS outer iteration, Jacobi / RAS / Mixed / RAS+AA solves.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_latency tools/fp64_latency.cu && \
  ./build/fp64_latency > gpurun_out/fp64_latency.json
timeout 1200 python tools/variants.py solve main hmin16 hmin32 hmin64 > gpurun_out/strip_height_solves.jsonl 2>&1
timeout 600 python tools/kbench.py > gpurun_out/kbench_4096.json 2>&1
timeout 1200 python tools/sweep_opts.py layered 4096 '[{"omega_v":0.6,"alpha_p":1.0},{"omega_v":0.6,"alpha_p":1.0,"smoother":2},{"omega_v":0.6,"alpha_p":1.0,"smoother":3},{"omega_v":0.6,"alpha_p":1.0,"smoother":2,"accel":2,"aa_depth":10,"aa_beta":1.0}]' > gpurun_out/ras_solves.jsonl 2>&1
cat gpurun_out/fp64_latency.json gpurun_out/strip_height_solves.jsonl gpurun_out/kbench_4096.json gpurun_out/ras_solves.jsonl
