#!/bin/bash
# A/B of attention variants on one box: quick C3 bench lines (no extras) with env switches.
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v"
  env $v timeout 600 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('value',d['value'],'gen',d['generation']['value'],'ms',d['ms_per_step'],'attn ms',d['kernels']['attention']['ms_per_step'],'frac',d['roofline']['frac'],'clk',d['clocks']['sm_mhz'])"
done
