# GEMM with 6 mainloop stages and a 4 KB epilogue staging ring per warp (-DB2S_GEMM_S6, plain
# epilogues only) vs the default 5 stages / 8 KB: plain-shape timings, then the layout / fp32 set
# (the B2S_GEMM_S6 #ifdef was removed after this measurement)
O=gpurun_out/r2s6; mkdir -p $O
for rep in 1 2; do for v in base s6; do
  if [ "$v" = base ]; then L=""; else L=paper_2602_08387_b200/csrc/build/var_$v/libb2s.so; fi
  for shp in "16384 8192 2048" "16384 2048 8192" "16384 3072 768" "16384 16384 2048"; do
    B2S_LIB=$L timeout 300 python tools/gemm_force_sweep.py $shp 2>/dev/null | head -1 | sed "s/^/$v $rep $shp /"
  done
  B2S_LIB=$L timeout 300 python tools/gemm_layout_ab.py 2>/dev/null | grep -v '"out": "bf16"' | sed "s/^/$v $rep /"
done; done
