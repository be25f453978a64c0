#!/bin/bash
# Sweep of scripts/kv_stream_bench.cu on a B200 (via gpurun): ring depths, page-table access, pool layout.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/kv_stream_bench.cu -o /tmp/kvb -lcuda || exit 1
for cfg in "2 2 0 0 0" "2 2 0 1 0" "2 2 0 0 1" "2 2 0 1 1" "3 2 0 1 0" "3 3 0 1 0" "4 3 0 1 0" "3 3 0 1 1" \
           "2 2 1500 0 0" "2 2 1500 1 0" "3 2 1500 1 0" "3 3 1500 1 0" "3 3 1500 1 1" "4 2 1500 1 0"; do
  timeout 60 /tmp/kvb $cfg 1280 512
done
