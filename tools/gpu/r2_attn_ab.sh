# A/B attention variants: bash tools/gpu/r2_attn_ab.sh name1 name2 ...  (default build = "base")
O=gpurun_out/r2attn_ab; mkdir -p $O
for rep in 1 2; do
for v in base "$@"; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  B2S_LIB=$L python tools/bench_attn.py gpt2-124m llama-1b llama-8b 2>/dev/null | grep '"b2s"' | sed "s/^/$v $rep /" >> $O/ab.txt
done
done
cat $O/ab.txt
