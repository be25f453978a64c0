# one GPU call: fresh per-kernel breakdown + GEMM shapes vs cuBLAS
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include scripts/gemm_bench.cu -o /tmp/gemm_bench -Lpaper_2601_23278_b200 -lfocus -Xlinker -rpath=$PWD/paper_2601_23278_b200 2>/dev/null || exit 1
for M in 428 728; do timeout 120 /tmp/gemm_bench $M; done > gpurun_out/gemm_bench.txt 2>&1
timeout 120 python scripts/cublas_ref.py 428 > gpurun_out/cublas.txt 2>&1
timeout 120 python scripts/cublas_ref.py 728 >> gpurun_out/cublas.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/gemm_bench.txt gpurun_out/cublas.txt; tail -c 3000 gpurun_out/bench.json
