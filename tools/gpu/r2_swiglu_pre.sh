# SwiGLU-backward GEMM with the first chunk's gate / up tiles issued before the accumulator wait,
# vs the default build: kernel timing x3, then GEMM / headline parity with the variant
O=gpurun_out/r2sgb; mkdir -p $O
for rep in 1 2 3; do
for v in base sgb; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  B2S_LIB=$L python tools/one_swiglu_bwd.py 2>/dev/null | sed "s/^/$v $rep /" >> $O/ab.txt
done
done
cat $O/ab.txt
B2S_LIB=paper_2602_08387_b200/csrc/build/var_sgb/libb2s.so timeout 600 python -m pytest tests/test_gemm.py tests/test_headline_parity.py -m gpu -q -x 2>&1 | tail -2
