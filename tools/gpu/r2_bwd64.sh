O=gpurun_out/r2bwd64; mkdir -p $O
timeout 300 python -m pytest tests/test_attn.py -q -x -m gpu > $O/test.log 2>&1; echo test $?; tail -3 $O/test.log
timeout 300 python tools/bench_attn.py gpt2-124m llama-1b 2>/dev/null | grep '"b2s"'
L=paper_2602_08387_b200/csrc/build/var_trace/libb2s.so
B2S_LIB=$L timeout 120 python tools/attn_bwd_trace.py 4 4096 32 8 > $O/trace.txt 2>&1; echo trace $?
