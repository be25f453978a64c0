#!/bin/bash
# GPU tests, smoke, the default C3 bench line, and the C3 ncu launch list + layer-10 --set full.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench C3 rc $?"
python scripts/profile_step.py C3 260 > gpurun_out/plain_step.log 2>&1 && bash scripts/gpu_suite.sh launches && bash scripts/gpu_suite.sh full
