#!/bin/bash
# End-of-session bench lines of the non-headline workloads (C2, C6, C3B64, C4) on one B200.
mkdir -p gpurun_out
for w in C2 C6 C3B64 C4; do
  timeout 1200 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "bench $w rc $?"
done
