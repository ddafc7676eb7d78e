# attention-backward prep kernel in [b, h, t] item order vs the default build: ncu durations of
# the prep launches at the 1B / 8B shapes, then the attention parity tests with the variant
O=gpurun_out/r2prep; mkdir -p $O
for v in base prep; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  B2S_LIB=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:attn_bwd_prep -c 6 --csv \
    python tools/bench_attn.py llama-1b llama-8b > $O/ncu_$v.csv 2>/dev/null
done
B2S_LIB=paper_2602_08387_b200/csrc/build/var_prep/libb2s.so timeout 600 python -m pytest tests/test_attn.py tests/test_headline_parity.py -m gpu -q -x 2>&1 | tail -2
