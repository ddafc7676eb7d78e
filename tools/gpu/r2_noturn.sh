L=paper_2602_08387_b200/csrc/build/var_noturn128/libb2s.so
B2S_LIB=$L timeout 600 python -m pytest tests/test_attn.py tests/test_headline_parity.py -k "attn or attention" -m gpu -q -x 2>&1 | tail -1
for i in 1 2; do
python tools/bench_attn.py llama-8b 2>/dev/null | grep '"b2s"' | grep fwd | sed 's/^/turns   /'
B2S_LIB=$L python tools/bench_attn.py llama-8b 2>/dev/null | grep '"b2s"' | grep fwd | sed 's/^/noturns /'
done
