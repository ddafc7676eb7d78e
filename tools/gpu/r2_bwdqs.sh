bash tools/gpu/r2_attn_test.sh
bash tools/gpu/r2_bwd_trace.sh
