python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/gemm_bench.cu -o /tmp/gemm_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200 2>/dev/null || exit 1
for M in 428 728; do timeout 120 /tmp/gemm_bench $M; done 2>&1 | grep -v check
GEMM_TRACE=1 timeout 60 /tmp/gemm_bench 428 > /dev/null 2>&1; python scripts/gemm_trace_report.py gpurun_out/gemm_trace_M428_*.bin 2>&1 | grep -E "bin|leaders"
