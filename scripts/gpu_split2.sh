python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/gemm_bench.cu -o /tmp/gemm_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200 2>/dev/null || exit 1
for M in 428 728; do timeout 60 /tmp/gemm_bench $M; FOCUS_GEMM_SPLIT2=0 GEMM_TAG=nosplit timeout 60 /tmp/gemm_bench $M; done 2>&1 | grep -E "M=|o\(|down"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
bash scripts/gpu_variants.sh "split2:" "nosplit:FOCUS_GEMM_SPLIT2=0" "split2b:"
