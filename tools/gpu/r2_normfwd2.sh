# norm forward (prefetch + 4 blocks/SM for D >= 2048 only) vs the default build: bench_ew norm
# lines, then the norm parity tests with the variant library
O=gpurun_out/r2nf2; mkdir -p $O
for rep in 1 2 3; do
for v in base nfx; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  B2S_LIB=$L python tools/bench_ew.py 2>/dev/null | grep norm_fwd | sed "s/^/$v $rep /" >> $O/ab.txt
done
done
cat $O/ab.txt
B2S_LIB=paper_2602_08387_b200/csrc/build/var_nfx/libb2s.so timeout 600 python -m pytest tests/test_ew.py tests/test_fp32_mode.py -m gpu -q -x 2>&1 | tail -2
