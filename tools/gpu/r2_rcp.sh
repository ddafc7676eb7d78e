# Approximate-reciprocal sigmoid in the SwiGLU epilogues + packed-fp32 forward softmax vs HEAD
# (.ab_base, tools/ab_base.sh): kernel A/B, GEMM / attention / SwiGLU parity, then step A/B
O=gpurun_out/r2rcp; mkdir -p $O
for i in 1 2; do
  for t in base new; do
    if [ $t = base ]; then D=.ab_base; else D=.; fi
    (cd $D && python tools/one_swiglu_bwd.py && python tools/one_swiglu_fwd.py) 2>/dev/null | sed "s/^/$t /" >> $O/kern.txt
  done
done
cat $O/kern.txt
timeout 900 python -m pytest tests/test_gemm.py tests/test_attn.py tests/test_headline_parity.py -m gpu -x -q > $O/test.log 2>&1; tail -2 $O/test.log
bash tools/gpu/ab_bench.sh
