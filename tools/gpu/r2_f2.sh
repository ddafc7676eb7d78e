# Packed-fp32 (FFMA2 / FADD2 / FMUL2) softmax and dS streams: attention parity with the variant
# library, then the same-box attention A/B (tools/gpu/r2_attn_ab.sh)
O=gpurun_out/r2f2; mkdir -p $O
B2S_LIB=paper_2602_08387_b200/csrc/build/var_f2/libb2s.so timeout 900 python -m pytest tests/test_attn.py -m gpu -x -q > $O/test.log 2>&1; tail -3 $O/test.log
bash tools/gpu/r2_attn_ab.sh f2
