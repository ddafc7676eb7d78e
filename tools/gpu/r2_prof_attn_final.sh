O=gpurun_out/r2pa; mkdir -p $O
timeout 300 python tools/bench_attn.py gpt2-124m llama-1b llama-8b > $O/bench_attn.jsonl 2>/dev/null; echo b $?
ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -s 2 -c 1 -o $O/attn_fwd_1b python tools/one_attn.py 4 4096 32 8 bwd > /dev/null 2>&1; echo a1 $?
DH=128 ncu --set full --import-source on --clock-control none -k regex:attn_bwd128_kernel -s 1 -c 1 -o $O/attn_bwd128_8b python tools/one_attn.py 2 4096 32 8 bwd > /dev/null 2>&1; echo a2 $?
DH=128 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_q_kernel -s 1 -c 1 -o $O/attn_bwdq128_8b python tools/one_attn.py 2 4096 32 8 bwd > /dev/null 2>&1; echo a3 $?
