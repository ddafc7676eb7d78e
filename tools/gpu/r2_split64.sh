timeout 600 python -m pytest tests/test_attn.py tests/test_headline_parity.py tests/test_guards.py -k "attn or attention" -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
(cd .ab_base && python tools/bench_attn.py gpt2-124m llama-1b 2>/dev/null | grep '"b2s"' | grep bwd | sed 's/^/base /')
python tools/bench_attn.py gpt2-124m llama-1b 2>/dev/null | grep '"b2s"' | grep bwd | sed 's/^/new  /'
done
