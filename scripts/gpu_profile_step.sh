# ncu evidence for the current tree (one C3 decode step): launch list + --set full of layer 2's GEMMs/attention
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
export FOCUS_NCU_STEP=1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu list rc $?"
# kernels matching the regex in step order: L0 qkv attn o gu down | L1 qkv importance | L1-suffix attn o gu down | L2 qkv attn o gu down
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_gemm_pair|k_attn_tc" -s 11 -c 5 -o gpurun_out/layer2_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
python scripts/ncu_summary.py gpurun_out/layer2_full.ncu-rep > gpurun_out/layer2_full_summary.txt 2>&1; head -90 gpurun_out/layer2_full_summary.txt
