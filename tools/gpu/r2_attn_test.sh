O=gpurun_out/r2attn_t; mkdir -p $O
timeout 600 python -m pytest tests/test_attn.py tests/test_headline_parity.py -k "attn" -m gpu -q -x > $O/test.log 2>&1; echo test $?
tail -3 $O/test.log
timeout 300 python tools/bench_attn.py gpt2-124m llama-1b llama-8b 2>/dev/null | grep '"b2s"' > $O/bench.txt; cat $O/bench.txt
