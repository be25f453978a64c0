python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
# skip prefill (64 req x 36 layers x 4 GEMMs = 9216) + warm-up step 1 (145) + layers 0,1 of step 2 (8): layer-2 QKV, O, GU, down
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 9369 -c 4 -o gpurun_out/gemm_prof python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1; echo "ncu rc $?"
