python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
# layer-2 GEMMs of decode step 2: skip prefill (64 x 36 x 4) + step 1 (145) + layers 0,1 of step 2 (8)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 9369 -c 4 -o gpurun_out/gemm_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc $?"
# layer-2 attention of decode step 2: skip prefill (64 x 36) + step 1 (37) + layer 0, importance, layer-1 suffix
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_tc -s 2344 -c 1 -o gpurun_out/attn_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1; echo "ncu attn rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 16300 -c 700 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc $?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
