python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/gemm_bench.cu -o /tmp/gemm_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200 2>/dev/null || exit 1
for M in 428 728; do
GEMM_TAG=bn256psk FOCUS_GEMM_BN256=1 FOCUS_GEMM_PSK=1 timeout 120 /tmp/gemm_bench $M
GEMM_TAG=psk FOCUS_GEMM_PSK=1 timeout 120 /tmp/gemm_bench $M
GEMM_TAG=bn256 FOCUS_GEMM_BN256=1 timeout 120 /tmp/gemm_bench $M
done 2>&1 | grep -v check
