#!/bin/bash
# Build and run the sweep-body microbenchmarks (design studies) on the GPU box.
set -u
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/body2_bench tools/body2_bench.cu && /tmp/body2_bench
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sweep_body_bench tools/sweep_body_bench.cu && /tmp/sweep_body_bench
