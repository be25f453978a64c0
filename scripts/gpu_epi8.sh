python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/gemm_bench.cu -o /tmp/gemm_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200 2>/dev/null || exit 1
for M in 428 728; do timeout 40 /tmp/gemm_bench $M; echo "gemm_bench rc $?"; done 2>&1 | grep -v "^status"
timeout 500 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 bash scripts/gpu_variants.sh "epi8:" "epi8b:"
