L=paper_2602_08387_b200/csrc/build/var_tracekv/libb2s.so
DH=128 B2S_LIB=$L python tools/attn_bwd_trace.py 2 4096 32 8 > gpurun_out/attn_bwdkv_trace_8b.txt 2>&1; echo $?
