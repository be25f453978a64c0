set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_base_pytest.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/r2_base_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_base_bench.json 2> gpurun_out/r2_base_bench.err; echo "bench rc $?"
tail -c 600 gpurun_out/r2_base_bench.json
