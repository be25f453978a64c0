python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/tma_bench.cu -o /tmp/tma_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200 2>/dev/null || exit 1
timeout 120 /tmp/tma_bench 2>&1 | tee gpurun_out/tma_bench.txt
