timeout 600 python -m pytest tests/test_attn.py tests/test_headline_parity.py tests/test_guards.py -m gpu -q -x -k "attn or attention" 2>&1 | tail -3
for i in 1 2; do
B2S_ATTN_FWD_V1=1 python tools/bench_attn.py gpt2-124m llama-1b 2>/dev/null | grep '"b2s"' | grep fwd | sed s/^/v1\ /
python tools/bench_attn.py gpt2-124m llama-1b 2>/dev/null | grep '"b2s"' | grep fwd | sed s/^/v4\ /
done
