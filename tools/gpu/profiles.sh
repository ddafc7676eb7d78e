# Regenerate the committed ncu evidence for the current code (one GPU; run each capture only
# after the same command exits 0 without ncu). Outputs land in gpurun_out/prof/, copied to
# profiles/ by hand.   bash tools/gpu/profiles.sh
set -x
O=gpurun_out/prof; mkdir -p $O
python tools/profile_step.py > $O/step_plain.log 2>&1 || exit 1
# 1. launch list of one GPT-2 step (serialised, cold-cache durations)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/gpt2_step_launches.csv \
    python tools/profile_step.py > $O/ncu1.log 2>&1
python tools/launch_table.py $O/gpt2_step_launches.csv > $O/gpt2_step_launches.txt
# 2. per-GEMM DRAM traffic + tensor-pipe activity over one step (bench.py's roofline "traffic")
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum \
    --clock-control none -k regex:gemm_kernel --csv --log-file $O/gemm_dram_tensor_metrics.csv \
    python tools/profile_step.py > $O/ncu2.log 2>&1
# 3. full captures of the top kernels
python tools/one_attn.py 8 2048 12 12 bwd > $O/attn.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:attn_fwd -c 1 -o $O/attn_fwd python tools/one_attn.py 8 2048 12 12 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -c 1 -o $O/attn_bwd python tools/one_attn.py 8 2048 12 12 bwd > /dev/null 2>&1
python tools/one_gelu_gemm.py 0 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 2 -c 1 -o $O/gemm_fc_fwd python tools/one_gelu_gemm.py 0 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 2 -c 1 -o $O/gemm_fc_fwd_gelu python tools/one_gelu_gemm.py 1 > /dev/null 2>&1
DH=128 python tools/one_attn.py 2 4096 32 8 bwd > $O/attn128.log 2>&1 && \
DH=128 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -c 1 -o $O/attn_fwd_dh128 python tools/one_attn.py 2 4096 32 8 > /dev/null 2>&1
ls -la $O
